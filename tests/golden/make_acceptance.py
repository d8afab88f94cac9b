"""Generates tests/golden/acceptance_c6c7.npz from the REFERENCE (oracle/_ref/libpcvref.so,
`pcvref_corrupted_run`: the shuffle-benchmark acceptance harness of acceptance.cpp:259-325 on the
reference's own ScoreAccum / rhat_from_blocks / shuffle_benchmark / benchmark_verdict).

    python tests/golden/make_acceptance.py

Per kind (0 clean with R = 500 replicates, criterion C6; 1 stuck chain and 2 +5 shift with R = 100,
criterion C7) and seed 0..19: the observed R-hat max, the 0.99 nearest-rank benchmark quantile and
the verdict. tests/test_gpu_acceptance.py feeds the same score streams (regenerated from the
bit-exact Philox streams) through pcvg_run_streams on the device and compares.
"""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(os.path.dirname(os.path.dirname(HERE)), "oracle", "_ref", "libpcvref.so")
BENCH_DRAWS = {0: 500, 1: 100, 2: 100}


def main():
    lib = C.CDLL(REF)
    f = lib.pcvref_corrupted_run
    f.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double),
                  C.POINTER(C.c_int32)]
    obs, qv, ok = np.zeros((3, 20)), np.zeros((3, 20)), np.zeros((3, 20), dtype=np.int32)
    o, q, p = C.c_double(), C.c_double(), C.c_int32()
    for kind in range(3):
        for seed in range(20):
            assert f(seed, kind, BENCH_DRAWS[kind], C.byref(o), C.byref(q), C.byref(p)) == 0
            obs[kind, seed], qv[kind, seed], ok[kind, seed] = o.value, q.value, p.value
    np.savez_compressed(os.path.join(HERE, "acceptance_c6c7.npz"), observed=obs, quantile_value=qv, verdict_pass=ok,
                        bench_draws=np.array([BENCH_DRAWS[k] for k in range(3)]))
    print("clean passes", ok[0].sum(), "/20; stuck flagged", 20 - ok[1].sum(), "/20; shift flagged", 20 - ok[2].sum(), "/20")


if __name__ == "__main__":
    main()

"""Wall-clock of one full-data fit (Step 1: adapt_full_data, 4 chains, 1,000 warm-up + 2,000 draws,
n_lf 32; engine.hpp:36-38) for a BASELINE config, on the device (pcvg_adapt_full_data) and with the
reference's own adapt_full_data (oracle/_ref, the unmodified reference library; the logistic family
runs as the oracle plugin on the reference engine) on the host cores - the "single full-data fit"
the north star compares the PCV run against.

  python tools/fit_time.py [--config cfg2] [--no-ref]

Test / measurement infrastructure: imports oracle/ only for the reference leg.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden"), os.path.join(ROOT, "tools")):
    sys.path.insert(0, p)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--no-ref", action="store_true")
    args = ap.parse_args()
    from bench_configs import CONFIGS, make_case
    from parity_util import Case
    from paper_2310_07002_b200 import pcv
    fixture, _, desc = CONFIGS[args.config]
    case = make_case(args.config)
    line = {"config": args.config, "workload": desc, "fit": "4 chains, 1000 warm-up + 2000 draws, n_lf 32"}
    with pcv.Context(0) as ctx:
        m = case.models[0]
        ctx.adapt_full_data(m, pcv.AdaptConfig(), seed=1, model_id=0)  # warm the context and the kernels
        t0 = time.perf_counter()
        f = ctx.adapt_full_data(m, pcv.AdaptConfig(), seed=2, model_id=0)
        line["device"] = {"wall_s": time.perf_counter() - t0, "device_s": f.device_ms / 1e3,
                          "step_size": f.kparams.step_size}
    if not args.no_ref:
        import _oracle as O
        from paper_2310_07002_b200 import abi
        if O.have_ref():
            rm = O.RModel(case.data, case.fa, abi.SpecArrays(**case.kws[0]))
            t0 = time.perf_counter()
            fit = rm.adapt(chains=4, warmup=1000, draws=2000, n_lf=32, seed=2)
            line["reference_cpu"] = {"wall_s": time.perf_counter() - t0, "step_size": fit["step_size"],
                                     "host_threads": os.cpu_count(),
                                     "kind": "reference adapt_full_data (oracle/_ref)"}
            line["reference_over_device"] = line["reference_cpu"]["wall_s"] / line["device"]["wall_s"]
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

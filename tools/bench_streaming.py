"""Throughput of the logistic path at the HBM-streaming size (tests/parity_util.StreamCase:
N = 400,000, P = 50, K-fold K = 1,184 x 8 chains = one 148-tile wave): the padded design matrix
(166 MB) exceeds the 126 MB L2, so every gradient pass streams X from HBM through the TMA ring.
Prints one JSON line: chain-steps/s, the FP64 DMMA fraction (algorithmic flops)
and the X bytes each pass must stream, i.e. the HBM rate the kernel needs at the measured speed.

  python tools/bench_streaming.py [--n 400000] [--folds 1184] [--steps 3] [--warmup 1]

Under ncu (one launch: --steps 1 --warmup 0) the capture gives the DRAM bytes per launch.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")):
    sys.path.insert(0, p)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=400_000)
    ap.add_argument("--folds", type=int, default=1184)
    ap.add_argument("--chains", type=int, default=8)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    args = ap.parse_args()
    from parity_util import StreamCase
    from paper_2310_07002_b200 import abi, pcv
    cs = StreamCase(args.n, args.folds)
    L = args.chains
    ctx = pcv.Context(0)
    ctx.add_model(cs.models[0], cs.kparams[0], cs.banks[0], model_id=0)
    cfg = abi.run_config(chains=L, iters=args.steps, warmup=args.warmup, batch_size=max(1, args.steps),
                         bench_draws=10, seed=1)
    ctx.begin(cfg)  # includes the warm-up iterations
    ms = []
    for _ in range(args.steps):
        ctx.advance(1)
        ms.append(ctx.last_advance_ms()[0])
    ctx.close()
    chains = cs.K * L
    n_lf = cs.kparams[0].n_leapfrog
    p1 = cs.data.x.shape[1] + 1
    value = chains * args.steps / (np.sum(ms) / 1e3)
    flop = n_lf * 4.0 * args.n * p1
    peak = json.load(open(os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")))["dmma_tflops_bps8"]
    sec_per_step = np.sum(ms) / 1e3 / args.steps
    x_bytes = args.n * (52 * 8 + 8 + 4)  # TMA tile bytes per row: X (52 padded columns), y, fold key
    tiles = (chains + 63) // 64
    line = {"workload": f"logistic N={args.n} P=50, K-fold K={cs.K} x {L} chains (one wave of {tiles} tiles), "
                        f"n_lf={n_lf}, FP64",
            "chains": chains, "steps": args.steps, "ms_per_step": sec_per_step * 1e3,
            "chain_steps_per_s": value, "flop_per_chain_step": flop,
            "achieved_tflops": flop * value / 1e12, "dmma_peak_tflops": peak,
            "frac_dmma": flop * value / 1e12 / peak,
            "x_bytes_per_pass": x_bytes, "x_exceeds_l2": x_bytes > 126e6,
            "x_stream_gbps_if_read_once_per_pass": x_bytes * n_lf / sec_per_step / 1e9,
            "x_stream_gbps_if_read_by_every_cta": x_bytes * n_lf * tiles / sec_per_step / 1e9}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

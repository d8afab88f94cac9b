"""Where the wall-clock of a converged PCV run goes: context creation, model upload (including the
host-built fold statistics), the run itself (device warm-up + sampling vs the rest: fold stats,
shuffle benchmark, report), and the same run again in the warm context.

  python tools/phase_times.py [--config cfg3] [--iters 1000] [--every 50]
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
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--every", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=100)
    args = ap.parse_args()
    from bench_configs import CONFIGS
    from parity_util import Case
    from paper_2310_07002_b200 import abi, pcv
    fixture, L, desc = CONFIGS[args.config]
    case = Case(fixture)
    cfg = abi.run_config(chains=L, iters=args.iters, warmup=args.warmup, batch_size=args.every, blocks=5,
                         bench_draws=500, seed=1, checkpoint_every=args.every, early_stop=1)
    out = {"config": args.config}
    t0 = time.perf_counter()
    ctx = pcv.Context(0)
    out["context_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    for i, (m, kp, bank) in enumerate(zip(case.models, case.kparams, case.banks)):
        ctx.add_model(m, kp, bank, model_id=i)
    out["add_models_s"] = time.perf_counter() - t0
    for tag in ("run_cold", "run_warm"):
        t0 = time.perf_counter()
        rep = ctx.run(cfg)
        wall = time.perf_counter() - t0
        dev = (rep["warmup_ms"] + rep["sampling_ms"]) / 1e3
        out[tag] = {"wall_s": wall, "sampler_device_s": dev, "rest_s": wall - dev, "iters_run": int(rep["iters_run"]),
                    "delta_hat": rep["delta_hat"]}
    ctx.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

"""Wall-clock to R-hat-converged elpd (the second half of BASELINE.json's metric): a full PCV run
with the early-stop rule (R-hat max within the 0.99 benchmark quantile and MCSE below
the epistemic SE, checked every `--every` iterations) through the public API, with host inputs.

  python tools/converge.py [--config cfg2] [--iters 1000] [--every 50]

Prints one JSON line: iterations run, wall-clock, device time, the elpd / delta and its errors,
and the reference CPU path's projected time for the same chain-steps (measured rate on a sample).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden"), os.path.join(ROOT, "tools")):
    sys.path.insert(0, p)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--every", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=100)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--device-fit", action="store_true",
                    help="run the PCV on the kernel and bank of a device Step 1 with the reference defaults "
                         "(4 chains, 1000 warm-up + 2000 draws; run_pcv_with_fits, engine.cpp:493-503) instead of "
                         "the fixture's reference-adapted kernel")
    ap.add_argument("--fit", action="store_true",
                    help="also time one full-data fit per model (Step 1, adapt_full_data defaults: "
                         "4 chains, 1000 warm-up + 2000 draws) on the same GPU, for the north star's "
                         "'comparable to a single full-data fit'")
    args = ap.parse_args()
    from bench_configs import CONFIGS, cpu_sample, make_case
    from parity_util import Case
    from paper_2310_07002_b200 import abi, pcv
    fixture, L, desc = CONFIGS[args.config]
    case = make_case(args.config)
    cfg = abi.run_config(chains=L, iters=args.iters, warmup=args.warmup, batch_size=args.every, blocks=5,
                         bench_draws=500, seed=1, checkpoint_every=args.every, early_stop=1)
    t0 = time.perf_counter()
    fit_s = 0.0
    if args.device_fit:
        fits = [pcv.adapt_full_data(m, pcv.AdaptConfig(), seed=1, model_id=i) for i, m in enumerate(case.models)]
        inputs = [pcv.ModelInput(m, f, i) for i, (m, f) in enumerate(zip(case.models, fits))]
        fit_s = time.perf_counter() - t0
    else:
        inputs = [pcv.ModelInput(m, pcv.FullDataFit(kp, bank), i)
                  for i, (m, kp, bank) in enumerate(zip(case.models, case.kparams, case.banks))]
    rep = pcv.run_pcv(inputs, cfg)
    wall = time.perf_counter() - t0
    chains = case.K * L * len(case.models)
    steps = rep["iters_run"] + args.warmup
    line = {"config": args.config, "workload": desc, "chains": chains, "iters_run": int(rep["iters_run"]),
            "warmup": args.warmup, "check_every": args.every, "max_iters": args.iters,
            "stopped_early": bool(rep["iters_run"] < args.iters), "wall_s": wall,
            "kernel": "device Step 1 (1000 + 2000, wall %.1f s incl. in wall_s)" % fit_s if args.device_fit
            else "fixture (reference adapt_full_data)",
            "device_s": (rep["warmup_ms"] + rep["sampling_ms"]) / 1e3,
            "delta_hat": rep["delta_hat"], "mcse": rep["mcse"], "epistemic_se": rep["epistemic_se"],
            "rhat_max": rep["rhat_max"], "verdict_quantile_value": rep["verdict_quantile_value"],
            "verdict_pass": int(rep["verdict_pass"]), "chain_steps": chains * steps}
    if "snapshots" in rep:  # per check interval: iters, delta_hat, mcse, epistemic_se, prob, ess, rhat_max
        line["snapshots"] = [[float(v) for v in row] for row in np.asarray(rep["snapshots"])]
    if args.fit:
        fits = []
        with pcv.Context(0) as ctx:
            for i, m in enumerate(case.models):
                t1 = time.perf_counter()
                f = ctx.adapt_full_data(m, pcv.AdaptConfig(), seed=1, model_id=i)
                fits.append({"wall_s": time.perf_counter() - t1, "device_s": f.device_ms / 1e3,
                             "step_size": f.kparams.step_size})
        line["full_data_fit"] = {"per_model": fits, "config": "4 chains, 1000 warm-up + 2000 draws, n_lf 32",
                                 "note": "Step 1 on the same GPU (pcvg_adapt_full_data), warm context"}
    if not args.no_cpu:
        threads = os.cpu_count() or 1
        rate, kind, sample = cpu_sample(case, L, 8, 3, threads)
        line["cpu"] = {"chain_steps_per_s": rate, "kind": kind, "cores": threads, "sample": sample,
                       "projected_s_same_chain_steps": chains * steps / rate}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

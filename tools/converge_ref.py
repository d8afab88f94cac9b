"""The early-stop rule applied to the reference CPU engine: the reference has no early
stop, so its time to R-hat-converged elpd is the wall-clock of a run_pcv to the first check interval
t at which its own report meets the rule (verdict pass on `blocks` blocks, MCSE < epistemic SE).
Runs the compiled reference (oracle/_ref) at t = every*blocks, every*(blocks+1), ... on all host
threads, with the same kernel, bank and seeds as tools/converge.py.

  python tools/converge_ref.py [--config cfg1] [--iters 1000] [--every 50] [--start T]
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
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--every", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=100)
    ap.add_argument("--start", type=int, default=0, help="first check point (default every * blocks)")
    args = ap.parse_args()
    from bench_configs import CONFIGS, make_case
    from parity_util import Case
    from paper_2310_07002_b200 import abi
    import _oracle as O
    fixture, L, desc = CONFIGS[args.config]
    case = make_case(args.config)
    models = [O.RModel(case.data, case.fa, abi.SpecArrays(**kw)) for kw in case.kws]
    kernels = [abi.KernelArrays(k.step_size, k.n_leapfrog, k.inv_mass_diag) for k in case.kparams]
    threads = os.cpu_count() or 1
    tried = []
    line = None
    t = args.start or args.every * 5
    while t <= args.iters:
        cfg = abi.run_config(chains=L, iters=t, warmup=args.warmup, batch_size=args.every, blocks=5, bench_draws=500,
                             seed=1)
        t0 = time.perf_counter()
        rep = O.run_pcv_ref(models, list(range(len(models))), kernels, case.banks, cfg, threads=threads)
        wall = time.perf_counter() - t0
        ok = bool(rep["verdict_pass"]) and rep["mcse"] < rep["epistemic_se"]
        tried.append({"iters": t, "wall_s": wall, "rhat_max": rep["rhat_max"],
                      "quantile_value": rep["verdict_quantile_value"], "pass": ok})
        line = {"config": args.config, "engine": "reference (oracle/_ref run_pcv)", "threads": threads,
                "iters_to_converge": t if ok else None, "wall_s": wall, "delta_hat": rep["delta_hat"],
                "mcse": rep["mcse"], "rhat_max": rep["rhat_max"], "tried": tried}
        if ok:
            break
        t += args.every
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

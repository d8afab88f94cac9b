"""Which folds hold R-hat max of a run, and why: per-fold R-hat, estimate and the fold's chains'
divergence counts for the worst folds (a stuck chain shows as a fold with one chain diverging on
most transitions, or with R-hat far above the rest).

  python tools/rhat_diag.py [--config cfg5] [--iters 1000] [--top 10]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden"), os.path.join(ROOT, "tools")):
    sys.path.insert(0, p)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=100)
    ap.add_argument("--top", type=int, default=10)
    ap.add_argument("--device-fit", action="store_true", help="kernel and bank from the device Step 1 (defaults)")
    args = ap.parse_args()
    from bench_configs import CONFIGS
    from parity_util import Case
    from paper_2310_07002_b200 import abi, pcv
    fixture, L, desc = CONFIGS[args.config]
    case = Case(fixture)
    with pcv.Context(0) as c:
        fits = []
        for i, m in enumerate(case.models):
            if args.device_fit:
                f = c.adapt_full_data(m, pcv.AdaptConfig(), seed=1, model_id=i)
                fits.append((f.kparams, f.draws))
            else:
                fits.append((case.kparams[i], case.banks[i]))
        for i, (m, (kp, bank)) in enumerate(zip(case.models, fits)):
            c.add_model(m, kp, bank, model_id=i)
        rep = c.run(abi.run_config(chains=L, iters=args.iters, warmup=args.warmup, batch_size=50, bench_draws=100,
                                   seed=1))
    K, nm = case.K, len(case.models)
    rh = rep["rhat"].reshape(nm, K)
    div = rep["divergences"].reshape(nm, K, L)
    q = np.nanquantile(rh, [0.5, 0.9, 0.99, 0.999], axis=1)
    out = {"config": args.config, "iters": args.iters, "device_fit": args.device_fit, "rhat_max": rep["rhat_max"],
           "verdict_quantile_value": rep["verdict_quantile_value"], "rhat_quantiles_50_90_99_999": q.T.tolist(),
           "divergent_transitions": int(div.sum()), "step_size": [float(k.step_size) for k, _ in fits], "worst": []}
    for m in range(nm):
        for k in np.argsort(-np.nan_to_num(rh[m], nan=-1))[: args.top]:
            out["worst"].append({"model": m, "fold": int(k), "rhat": float(rh[m, k]),
                                 "estimate": float(rep["estimate"][m * K + k]), "divergences": div[m, k].tolist()})
    print(json.dumps(out))


if __name__ == "__main__":
    main()

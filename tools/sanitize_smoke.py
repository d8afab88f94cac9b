"""Small runs of the round-2 device paths for compute-sanitizer (memcheck / racecheck):
the lean kernel (cfg1 warm-up + sampling), the few-chain multi-cluster GLM launch (cfg2, one tile),
score-stream runs with early stop, fault injection, and the in-process multi-device driver.

  compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")):
    sys.path.insert(0, p)

from paper_2310_07002_b200 import abi, pcv  # noqa: E402
from parity_util import Case, sample_thetas  # noqa: E402


def main():
    c1 = Case("cfg1_linreg_loo")
    with pcv.Context(0) as c:
        c.add_model(c1.models[0], c1.kparams[0], c1.banks[0], model_id=0)
        c.debug_break_fold(0, 3)
        rep = c.run(abi.run_config(chains=4, iters=20, warmup=4, batch_size=5, bench_draws=10, seed=1,
                                   checkpoint_every=5, early_stop=1, blocks=2))
        print("lean run", rep["iters_run"], rep["delta_hat"])
    c2 = Case("cfg2_logistic_bench")
    with pcv.Context(0) as c:
        kp = c2.kparams[0]
        c.add_model(c2.models[0], pcv.KernelParams(kp.step_size, 2, kp.inv_mass_diag), c2.banks[0], model_id=0)
        th = sample_thetas(c2, 0, 20, seed=1)
        folds = np.arange(20, dtype=np.int32)
        lp, g = c.eval(0, folds, th)
        q, p, ok = c.leapfrog(0, folds, th, np.ones_like(th))
        print("multi-cluster eval / leapfrog", np.isfinite(lp).all(), ok.all())
    with pcv.Context(0) as c:
        s = np.random.default_rng(0).standard_normal((4, 3, 40))
        rep = c.run_streams(s, np.zeros(4), abi.run_config(chains=3, iters=40, batch_size=5, blocks=2, bench_draws=10,
                                                            checkpoint_every=10, early_stop=1, seed=2))
        print("streams", rep["iters_run"], rep["verdict_pass"])
    with pcv.MultiContext([0, 0]) as mc:
        mc.add_model(c1.models[0], c1.kparams[0], c1.banks[0], model_id=0)
        rep = mc.run(abi.run_config(chains=4, iters=20, warmup=4, batch_size=5, bench_draws=10, seed=1))
        print("multi-device", rep["delta_hat"])


if __name__ == "__main__":
    main()

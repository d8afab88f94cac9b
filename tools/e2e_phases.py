"""Where the bench's e2e wall-clock goes beyond the device sampler time (cfg2, bench sizes):
context + model upload, and run_pcv's own phases (device warm-up + sampling vs the rest)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")):
    sys.path.insert(0, p)
import torch  # noqa: E402  (the bench process has torch's context up before e2e)

from paper_2310_07002_b200 import pcv  # noqa: E402
from parity_util import Case  # noqa: E402

torch.zeros(1, device="cuda")
case = Case("cfg2_logistic_bench")
for rep_i in range(2):
    t0 = time.perf_counter()
    ctx = pcv.Context(0)
    t1 = time.perf_counter()
    ctx.add_model(case.models[0], case.kparams[0], case.banks[0], model_id=0)
    t2 = time.perf_counter()
    rep = ctx.run(pcv.RunConfig(chains=8, iters=10, warmup=3, batch_size=10, blocks=5, bench_draws=100, seed=1))
    t3 = time.perf_counter()
    ctx.close()
    t4 = time.perf_counter()
    dev = (rep["warmup_ms"] + rep["sampling_ms"]) / 1e3
    print(f"pass {rep_i}: context {t1 - t0:.3f} s, add_model {t2 - t1:.3f} s, run {t3 - t2:.3f} s "
          f"(sampler device {dev:.3f} s, rest {t3 - t2 - dev:.3f} s), close {t4 - t3:.3f} s", flush=True)

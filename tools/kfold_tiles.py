"""Few-chain logistic (cfg2 K-fold) per-iteration time vs chains per fold: one 64-chain tile
(L = 4 -> 40 chains) vs two (L = 8 -> 80 chains), to see whether the tiles' clusters overlap."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden"), os.path.join(ROOT, "tools")):
    sys.path.insert(0, p)
from bench_configs import gpu_run  # noqa: E402
from parity_util import Case  # noqa: E402
from paper_2310_07002_b200 import pcv  # noqa: E402

case = Case("cfg2_logistic_bench")
case.folds = pcv.make_kfold_scheme(case.data, 10, 1)
case.models = [pcv.LogisticModel("M0", case.data, case.folds)]
case.fa = case.folds.arrays()
for L in (4, 6, 8, 12):
    ms, _ = gpu_run(case, L, 3, 2)
    print(f"L={L}: {10 * L} chains, {ms / 3:.3f} ms per iteration", flush=True)

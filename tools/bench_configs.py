"""Per-configuration throughput for every BASELINE.json config on one B200, with the reference CPU
engine timed beside it on a bounded fold sample (same inputs: reference-adapted kernels and banks
from tests/golden/*). One JSON line per config.

  python tools/bench_configs.py [--steps K] [--warmup W] [--only cfg3,cfg4]

FLOPs per chain-step are the kernels' algorithmic counts (DESIGN.md 4.1/4.2):
  logistic: n_lf * 4 N (P+1);  Gaussian families: n_lf * N * (4 nc + 4)  (nc covariates read).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")):
    sys.path.insert(0, p)

CONFIGS = {
    "cfg1": ("cfg1_linreg_loo", 4, "linear regression N=100 P=5 (grouped, J=1), LOO 100 folds x 4 chains"),
    "cfg2": ("cfg2_logistic_bench", 8, "logistic N=10000 P=50, LOO 10000 folds x 8 chains"),
    "cfg2k": ("cfg2_logistic_bench", 8, "logistic N=10000 P=50, K-fold K=10 (seed 1) x 8 chains"),
    "cfg4r": ("cfg4_seasonal_bench", 4, "seasonal AR(2)+11 dummies T=5000, hv-block Racine per-point folds "
                                        "(K=4998, v=5, h=12), M_A+M_B x 4 chains"),
    "cfg3": ("cfg3_radon_bench", 8, "radon-style 12000 houses / 400 counties, LOGO, M_A+M_B x 8 chains"),
    "cfg4": ("cfg4_seasonal_bench", 4, "seasonal AR(2)+11 dummies T=5000, hv-block K=100 h=12, M_A+M_B x 4 chains"),
    "cfg5": ("cfg5_linreg_bench", 16, "linear regression N=100000 P=5, LOO 100000 folds x 16 chains"),
}


def make_case(name):
    """The test fixture of a config with its fold scheme: cfg2k is BASELINE configs[1]'s K-fold scheme
    on the cfg2 data and fit, cfg4r SURVEY 8(d)'s Racine per-point hv folds on the cfg4 data and fits."""
    from parity_util import Case
    fixture, _, _ = CONFIGS[name]
    case = Case(fixture)
    if name == "cfg2k":
        from paper_2310_07002_b200 import pcv
        case.folds = pcv.make_kfold_scheme(case.data, 10, 1)
        case.models = [pcv.LogisticModel("M0", case.data, case.folds)]
        case.fa = case.folds.arrays()
    if name == "cfg4r":
        from paper_2310_07002_b200 import pcv
        case.folds = pcv.make_hv_racine_scheme(case.data, 5, 12)
        case.models = [pcv.SeasonalARModel(f"M{m}", case.data, case.folds, kw["ar_order"], kw["dummies"],
                                           kw["rho_transform"]) for m, kw in enumerate(case.kws)]
        case.fa = case.folds.arrays()
    return case


def flops_per_chain_step(case, m):
    kw = case.kws[m]
    n = case.data.n_obs
    n_lf = case.kparams[m].n_leapfrog
    fam = kw["family"]
    from paper_2310_07002_b200 import abi
    if fam == abi.FAMILY_LOGISTIC:
        return n_lf * 4.0 * n * case.data.x.shape[1] + n_lf * 4.0 * n
    nc = {abi.FAMILY_GROUPED: case.data.x.shape[1], abi.FAMILY_RADON: 1,
          abi.FAMILY_SEASONAL_AR: kw["ar_order"] + kw["dummies"]}[fam]
    return n_lf * n * (4.0 * nc + 4.0)


def gpu_run(case, L, steps, warmup, policy=0):
    from paper_2310_07002_b200 import abi, pcv
    ctx = pcv.Context(0)
    ctx.set_kernel_policy(policy)
    for i, (m, kp, bank) in enumerate(zip(case.models, case.kparams, case.banks)):
        ctx.add_model(m, kp, bank, model_id=i)
    cfg = abi.run_config(chains=L, iters=steps, warmup=warmup, batch_size=min(50, steps), bench_draws=10, seed=1)
    ctx.begin(cfg)
    ms = []
    for _ in range(steps):
        ctx.advance(1)
        ms.append(ctx.last_advance_ms()[0])
    cols, _, _, done = ctx.fold_stats(case.K)
    ctx.close()
    return float(np.sum(ms)), cols


def cpu_sample(case, L, folds_sample, steps, threads):
    import ctypes as C
    import _oracle as O
    from paper_2310_07002_b200 import abi
    rng = np.random.default_rng(0)
    folds = np.sort(rng.choice(case.K, min(folds_sample, case.K), replace=False)).astype(np.int32)
    total = 0.0
    chain_steps = 0
    kind = "reference" if O.have_ref() else "port"
    for m in range(len(case.models)):
        kp = case.kparams[m]
        kern = abi.KernelArrays(kp.step_size, kp.n_leapfrog, kp.inv_mass_diag)
        bank = np.ascontiguousarray(case.banks[m])
        s_s, w_s, cs = C.c_double(), C.c_double(), C.c_double()
        spec = abi.SpecArrays(**case.kws[m])
        ref_ok = case.folds.intervals is None or case.kws[m]["family"] == abi.FAMILY_SEASONAL_AR
        if kind == "reference" and ref_ok:
            mod = O.RModel(case.data, case.fa, spec)
            fn = O.ref().pcvref_time_tasks
        else:
            mod = O.OModel(case.data, case.fa, spec)
            fn = O.oracle().pcvo_time_tasks
            kind = "port"
        rc = fn(mod.h, len(folds), abi.ptr(folds, C.c_int32), L, 1, steps, 1, m, C.byref(kern.struct),
                abi.ptr(bank, C.c_double), bank.shape[0], threads, C.byref(s_s), C.byref(w_s), C.byref(cs))
        assert rc == 0
        total += s_s.value
        chain_steps += len(folds) * L * steps
    return chain_steps / total, kind, f"{len(folds)} folds x {L} chains x {steps} steps x {len(case.models)} model(s)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--only", default="")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--policy", type=int, default=0, help="0 auto, 1 generic kernel, 2 tensor-core kernel, 4 fold sufficient statistics, 5 row-streaming kernels")
    args = ap.parse_args()
    from parity_util import Case
    peak = json.load(open(os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")))
    names = [n for n in CONFIGS if not args.only or n in args.only.split(",")]
    for name in names:
        fixture, L, desc = CONFIGS[name]
        case = make_case(name)
        steps = args.steps if name != "cfg5" else max(2, args.steps // 3)
        ms, cols = gpu_run(case, L, steps, args.warmup, args.policy)
        chains = case.K * L * len(case.models)
        value = chains * steps / (ms / 1e3)
        flops = sum(flops_per_chain_step(case, m) for m in range(len(case.models))) / len(case.models)
        achieved = flops * value / 1e12
        is_logistic = name.startswith("cfg2")
        pk = peak["dmma_tflops_bps8"] if is_logistic else peak["dfma_tflops_bps8"]
        # AUTO / SUFFSTAT run the Gaussian families on fold sufficient statistics: the
        # row-streaming flop count is then a row-equivalent rate, not a roofline fraction
        suff = not is_logistic and args.policy in (0, 4)
        line = {"config": name, "policy": args.policy, "kernel": "suffstat" if suff else "rows",
                "workload": desc, "chains": chains, "steps": steps,
                "gpu_chain_steps_per_s": value, "gpu_ms_per_step": ms / steps,
                "flop_per_chain_step": flops,
                ("row_equivalent_tflops" if suff else "achieved_tflops"): achieved,
                "peak_tflops": pk, "peak_kind": "FP64 DMMA" if is_logistic else "FP64 DFMA",
                "frac": None if suff else achieved / pk, "elpd_sum_model0": float(np.sum(cols["estimate"][:case.K]))}
        if not args.no_cpu:
            threads = os.cpu_count() or 1
            sample_folds = {"cfg1": 32, "cfg2": 32, "cfg2k": 2, "cfg3": 8, "cfg4": 8, "cfg4r": 8, "cfg5": 4}[name]
            cv, kind, sample = cpu_sample(case, L, sample_folds, 3, threads)
            line["cpu"] = {"chain_steps_per_s": cv, "kind": kind, "cores": threads, "sample": sample}
            line["speedup_vs_cpu"] = value / cv
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

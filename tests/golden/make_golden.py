"""Generates the committed golden fixtures under tests/golden/ from the REFERENCE itself.

Run here (needs /root/reference compiled into oracle/_ref/libpcvref.so by `make -C oracle ref`):
    python tests/golden/make_golden.py [name ...]

For every parity configuration it stores (npz): the dataset (from the product simulators, whose
bit-exactness against the reference simulators is a separate test), the fold assignment, the
reference's adapt_full_data kernel (step size + inverse mass) and draw bank per model
(adapt.cpp:96-221, the `_bank.f64` content), and the reference run_pcv report on that input
(engine.cpp:257-483). The GPU box has no /root/reference: GPU tests and bench.py read these files.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2310_07002_b200 import abi, pcv  # noqa: E402
import _oracle as O  # noqa: E402

# name -> (builder, models[(family spec kwargs)], adapt settings, run settings)


def _cfg1():
    d = pcv.simulate_linreg(100, 5, seed=11)
    f = pcv.make_loo_scheme(d)
    return d, f, [dict(family=abi.FAMILY_GROUPED)]


def _ex1():
    d = pcv.simulate_grouped_regression(50, 5, 4, 1.0, seed=1)
    f = pcv.make_logo_scheme(d)
    return d, f, [dict(family=abi.FAMILY_GROUPED, covariate_mask=[1, 1, 1, 1]),
                  dict(family=abi.FAMILY_GROUPED, covariate_mask=[1, 1, 1, 0])]


def _radon():
    d = pcv.simulate_radon_style(1200, 40, 5)
    f = pcv.make_logo_scheme(d)
    return d, f, [dict(family=abi.FAMILY_RADON, include_floor=1),
                  dict(family=abi.FAMILY_RADON, include_floor=0)]


def _seasonal_tb():
    d = pcv.simulate_seasonal_ar(600, 2, 11, 0.6, seed=7)
    f = pcv.make_time_block_scheme(d, 20)
    return d, f, [dict(family=abi.FAMILY_SEASONAL_AR, ar_order=2, dummies=11),
                  dict(family=abi.FAMILY_SEASONAL_AR, ar_order=2, dummies=0)]


def _seasonal_hv():
    d = pcv.simulate_seasonal_ar(600, 2, 11, 0.6, seed=7)
    f = pcv.make_hv_block_scheme(d, 20, 6)
    return d, f, [dict(family=abi.FAMILY_SEASONAL_AR, ar_order=2, dummies=11)]


def _rat():  # paper Ex-2 style: 30 rats x 5 weights, leave-one-subject-out, M_A vs M_B
    d = pcv.simulate_rat_growth(30, seed=4)
    f = pcv.make_logo_scheme(d)
    return d, f, [dict(family=abi.FAMILY_RAT_GROWTH, per_subject_slope=1),
                  dict(family=abi.FAMILY_RAT_GROWTH, per_subject_slope=0)]


def _logistic():
    d = pcv.simulate_logistic(500, 10, seed=1)
    f = pcv.make_loo_scheme(d)
    return d, f, [dict(family=abi.FAMILY_LOGISTIC)]


def _logistic_kfold():
    d = pcv.simulate_logistic(500, 10, seed=1)
    f = pcv.make_kfold_scheme(d, 10, 1)
    return d, f, [dict(family=abi.FAMILY_LOGISTIC)]


def _cfg2_bench():
    d = pcv.simulate_logistic(10000, 50, seed=1)
    f = pcv.make_loo_scheme(d)
    return d, f, [dict(family=abi.FAMILY_LOGISTIC)]


def _cfg3_bench():
    d = pcv.simulate_radon_style(12000, 400, 5)
    f = pcv.make_logo_scheme(d)
    return d, f, [dict(family=abi.FAMILY_RADON, include_floor=1),
                  dict(family=abi.FAMILY_RADON, include_floor=0)]


def _cfg4_bench():
    d = pcv.simulate_seasonal_ar(5000, 2, 11, 0.6, seed=7)
    f = pcv.make_hv_block_scheme(d, 100, 12)
    return d, f, [dict(family=abi.FAMILY_SEASONAL_AR, ar_order=2, dummies=11),
                  dict(family=abi.FAMILY_SEASONAL_AR, ar_order=2, dummies=0)]


def _cfg5_bench():
    d = pcv.simulate_linreg(100000, 5, seed=11)
    f = pcv.make_loo_scheme(d)
    return d, f, [dict(family=abi.FAMILY_GROUPED)]


# Bench fixtures store the simulator call instead of the data (regenerated bit-exactly).
SIM = {
    "cfg2_logistic_bench": ("logistic", [10000, 50, 1]),
    "cfg3_radon_bench": ("radon", [12000, 400, 5]),
    "cfg4_seasonal_bench": ("seasonal", [5000, 2, 11, 7]),
    "cfg5_linreg_bench": ("linreg", [100000, 5, 11]),
}


def _regenerate(kind, a):
    if kind == "logistic":
        d = pcv.simulate_logistic(a[0], a[1], seed=a[2])
        return d, pcv.make_loo_scheme(d)
    if kind == "radon":
        d = pcv.simulate_radon_style(a[0], a[1], a[2])
        return d, pcv.make_logo_scheme(d)
    if kind == "seasonal":
        d = pcv.simulate_seasonal_ar(a[0], a[1], a[2], 0.6, seed=a[3])
        return d, pcv.make_hv_block_scheme(d, 100, 12)
    d = pcv.simulate_linreg(a[0], a[1], seed=a[2])
    return d, pcv.make_loo_scheme(d)


CONFIGS = {
    # name: (builder, adapt kwargs, run kwargs or None)
    "cfg1_linreg_loo": (_cfg1, dict(chains=4, warmup=1000, draws=500), dict(chains=4, iters=200, warmup=50, batch_size=20, bench_draws=50, checkpoint_every=100)),
    "ex1_grouped_logo": (_ex1, dict(chains=4, warmup=1000, draws=250), dict(chains=4, iters=200, warmup=50, batch_size=20, bench_draws=50, checkpoint_every=100)),
    "radon_logo": (_radon, dict(chains=4, warmup=600, draws=250), dict(chains=4, iters=100, warmup=20, batch_size=10, bench_draws=50)),
    "seasonal_timeblocks": (_seasonal_tb, dict(chains=4, warmup=600, draws=250), dict(chains=4, iters=100, warmup=20, batch_size=10, bench_draws=50)),
    "seasonal_hvblock": (_seasonal_hv, dict(chains=4, warmup=600, draws=250), dict(chains=4, iters=100, warmup=20, batch_size=10, bench_draws=50)),
    "rat_logo": (_rat, dict(chains=4, warmup=1000, draws=250), dict(chains=4, iters=200, warmup=50, batch_size=20, bench_draws=50, checkpoint_every=100)),
    "logistic_loo": (_logistic, dict(chains=4, warmup=600, draws=250), dict(chains=4, iters=100, warmup=20, batch_size=10, bench_draws=50)),
    "logistic_kfold": (_logistic_kfold, dict(chains=4, warmup=600, draws=250), dict(chains=4, iters=100, warmup=20, batch_size=10, bench_draws=50)),
    # bench input only (no reference run: 80k chains is the GPU workload)
    "cfg2_logistic_bench": (_cfg2_bench, dict(chains=4, warmup=300, draws=250), None),
    "cfg3_radon_bench": (_cfg3_bench, dict(chains=4, warmup=400, draws=25), None),
    "cfg4_seasonal_bench": (_cfg4_bench, dict(chains=4, warmup=400, draws=25), None),
    "cfg5_linreg_bench": (_cfg5_bench, dict(chains=4, warmup=300, draws=25), None),
}


def make(name):
    builder, akw, rkw = CONFIGS[name]
    d, f, specs = builder()
    if name in SIM:
        kind, args = SIM[name]
        out = {"K": np.int64(f.K), "sim_kind": np.array(kind), "sim_args": np.array(args, dtype=np.int64)}
    else:
        out = {"y": d.y, "x": d.x, "K": np.int64(f.K)}
        if d.group_id is not None:
            out["group_id"] = d.group_id
        if d.time_index is not None:
            out["time_index"] = d.time_index
        if f.test_index is not None:
            out["test_index"] = f.test_index
        if f.intervals is not None:
            out["intervals"] = f.intervals
    fa = f.arrays()
    rmodels, kernels, banks = [], [], []
    for m, s in enumerate(specs):
        sa = abi.SpecArrays(**s)
        rm = O.RModel(d, fa, sa)
        fit = rm.adapt(seed=1, model_id=m, **akw)
        out[f"spec{m}"] = np.array([s.get("family"), s.get("include_floor", 1), s.get("ar_order", 1),
                                    s.get("dummies", 0), s.get("rho_transform", 0),
                                    s.get("per_subject_slope", 0)], dtype=np.int64)
        if s.get("covariate_mask") is not None:
            out[f"mask{m}"] = np.array(s["covariate_mask"], dtype=np.int32)
        out[f"step{m}"] = np.float64(fit["step_size"])
        out[f"inv_mass{m}"] = fit["inv_mass_diag"]
        out[f"bank{m}"] = fit["bank"]
        out[f"mean_accept{m}"] = np.float64(fit["mean_accept"])
        rmodels.append(rm)
        kernels.append(abi.KernelArrays(fit["step_size"], 32, fit["inv_mass_diag"]))
        banks.append(fit["bank"])
        print(f"  {name} model {m}: step {fit['step_size']:.4g} accept {fit['mean_accept']:.3f} "
              f"divergences {fit['divergences']}", flush=True)
    out["n_models"] = np.int64(len(specs))
    if rkw is not None:
        cfg = abi.run_config(seed=1, **rkw)
        rep = O.run_pcv_ref(rmodels, list(range(len(specs))), kernels, banks, cfg, threads=0)
        for k in ("delta_hat", "mcse", "sigma2_delta", "epistemic_se", "prob_a_better", "ess_overall",
                  "rhat_max", "dropped_batch_draws", "verdict_pass", "verdict_quantile_value"):
            out[f"ref_{k}"] = np.float64(rep[k])
        for k in ("estimate", "log_f_hat", "mc_contribution", "ess", "rhat", "batches", "fault",
                  "failed", "divergences", "delta_k", "snapshots", "benchmark"):
            out[f"ref_{k}"] = rep[k]
        out["ref_score_total"] = np.array(rep["score_total"])
        out["run_cfg"] = np.array([rkw["chains"], rkw["iters"], rkw["warmup"], rkw["batch_size"], 5,
                                   rkw["bench_draws"], rkw.get("checkpoint_every", 0)], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def load(name):
    """Loads a fixture into product descriptors: (data, folds, [(spec kwargs, KernelParams, bank)], npz)."""
    z = np.load(os.path.join(HERE, f"{name}.npz"))
    if "sim_logistic" in z:
        n, p, seed = (int(v) for v in z["sim_logistic"])
        d = pcv.simulate_logistic(n, p, seed=seed)
        f = pcv.make_loo_scheme(d)
    elif "sim_kind" in z:
        d, f = _regenerate(str(z["sim_kind"]), [int(v) for v in z["sim_args"]])
    else:
        d = pcv.Dataset(z["y"], z["x"], z["group_id"] if "group_id" in z else None,
                        z["time_index"] if "time_index" in z else None)
        f = pcv.FoldAssignment(int(z["K"]), z["test_index"] if "test_index" in z else None,
                               z["intervals"] if "intervals" in z else None)
    models = []
    for m in range(int(z["n_models"])):
        sp = [int(v) for v in z[f"spec{m}"]]
        fam, floor, p, q, rho = sp[:5]
        kw = dict(family=fam, include_floor=floor, ar_order=p, dummies=q, rho_transform=rho)
        if fam == abi.FAMILY_RAT_GROWTH:
            kw["per_subject_slope"] = sp[5]
        if f"mask{m}" in z:
            kw["covariate_mask"] = z[f"mask{m}"]
        kp = pcv.KernelParams(float(z[f"step{m}"]), 32, z[f"inv_mass{m}"])
        models.append((kw, kp, z[f"bank{m}"]))
    return d, f, models, z


# HS / DSS reference reports (engine.cpp:322-373, scoring.cpp:64-104) on the inputs of a base
# fixture: tests/golden/<base>_<hs|dss>.npz holds only the reference report for that score.
SCORE_FIXTURES = {
    "cfg1_linreg_loo": (abi.SCORE_HS, abi.SCORE_DSS),
    "ex1_grouped_logo": (abi.SCORE_HS, abi.SCORE_DSS),
    "radon_logo": (abi.SCORE_HS, abi.SCORE_DSS),
    "seasonal_timeblocks": (abi.SCORE_HS, abi.SCORE_DSS),
    "seasonal_hvblock": (abi.SCORE_HS, abi.SCORE_DSS),
    "rat_logo": (abi.SCORE_HS, abi.SCORE_DSS),
}
SCORE_NAME = {abi.SCORE_HS: "hs", abi.SCORE_DSS: "dss"}


def score_run_config(z, score):
    rc = z["run_cfg"]
    return abi.run_config(chains=int(rc[0]), iters=int(rc[1]), warmup=int(rc[2]), batch_size=int(rc[3]),
                          blocks=int(rc[4]), bench_draws=int(rc[5]), checkpoint_every=int(rc[6]), seed=1,
                          score=score)


def make_score(base, score):
    d, f, models, z = load(base)
    fa = f.arrays()
    rmodels = [O.RModel(d, fa, abi.SpecArrays(**kw)) for kw, _, _ in models]
    kernels = [abi.KernelArrays(kp.step_size, kp.n_leapfrog, kp.inv_mass_diag) for _, kp, _ in models]
    cfg = score_run_config(z, score)
    rep = O.run_pcv_ref(rmodels, list(range(len(models))), kernels, [b for _, _, b in models], cfg, threads=0)
    out = {"score": np.int64(score)}
    for k in ("delta_hat", "mcse", "sigma2_delta", "epistemic_se", "prob_a_better", "ess_overall",
              "rhat_max", "dropped_batch_draws", "verdict_pass", "verdict_quantile_value"):
        out[f"ref_{k}"] = np.float64(rep[k])
    for k in ("estimate", "log_f_hat", "mc_contribution", "ess", "rhat", "batches", "fault",
              "failed", "dss_ridged", "divergences", "delta_k", "snapshots", "benchmark"):
        out[f"ref_{k}"] = rep[k]
    out["ref_score_total"] = np.array(rep["score_total"])
    np.savez_compressed(os.path.join(HERE, f"{base}_{SCORE_NAME[score]}.npz"), **out)


# Short full-data adaptations by the reference (adapt.cpp:96-221) on fixture inputs, short enough
# that the device run follows the same chain trajectories: tests/golden/adapt_short.npz.
ADAPT_SHORT = dict(chains=4, warmup=30, draws=10, n_lf=32)
ADAPT_BASES = ["cfg1_linreg_loo", "ex1_grouped_logo", "radon_logo", "seasonal_timeblocks",
               "seasonal_hvblock", "logistic_loo", "rat_logo"]


def make_adapt_short():
    out = {}
    for base in ADAPT_BASES:
        d, f, models, z = load(base)
        fa = f.arrays()
        for m, (kw, _, _) in enumerate(models):
            rm = O.RModel(d, fa, abi.SpecArrays(**kw))
            fit = rm.adapt(seed=3, model_id=m, **ADAPT_SHORT)
            out[f"{base}:{m}:step"] = np.float64(fit["step_size"])
            out[f"{base}:{m}:inv_mass"] = fit["inv_mass_diag"]
            out[f"{base}:{m}:bank"] = fit["bank"]
            out[f"{base}:{m}:accept"] = np.float64(fit["mean_accept"])
            out[f"{base}:{m}:div"] = np.int64(fit["divergences"])
            if m == 0:  # per-iteration traces of the restated loop (ref_shim pcvref_adapt_trace)
                tr = rm.adapt_trace(chains=4, warmup=30, seed=3, model_id=m)
                out[f"{base}:{m}:init_step"] = np.float64(tr["init_step"])
                out[f"{base}:{m}:step_trace"] = tr["step_trace"]
                out[f"{base}:{m}:ap_trace"] = tr["ap_trace"]
    np.savez_compressed(os.path.join(HERE, "adapt_short.npz"), **out)


if __name__ == "__main__":
    names = sys.argv[1:] or list(CONFIGS) + ["scores", "adapt"]
    for nm in names:
        print(nm, flush=True)
        if nm == "adapt":
            make_adapt_short()
        elif nm == "scores":
            for base, scores in SCORE_FIXTURES.items():
                for sc in scores:
                    make_score(base, sc)
        else:
            make(nm)

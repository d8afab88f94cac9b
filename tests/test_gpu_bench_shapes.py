"""GPU parity at the BASELINE shapes the bench and the convergence runs actually use (SURVEY 8(c)
protocol (2)-(4); the fixtures of test_gpu_parity.py are small). Every probe goes through the C ABI.

* cfg2 (bench.py's workload): logistic N=10,000, P=50 -> glm_kernel<logistic,52> (64-row TMA tiles,
  KS=13, PT=7). Probed with enough chains for full 148-tile waves plus a wave tail (the tail runs as
  row-split clusters) and with a single 64-chain tile (16-CTA cluster, the few-chain geometry).
  Log joint / gradient / log_pred / injected hmc_step and leapfrog end points with n_leapfrog = 1
  (the precise value pass only) and 2 (one gradient-only pass with the fast sigmoid,
  tc_common.cuh::logistic_resid_fast), all at 1e-12 of the sum of absolute terms (hmc.cpp:22-99).
* cfg4: seasonal AR T=5,000 (4,998 rows), hv-block K=100, h=12, both models, on the
  sufficient-statistics kernel and on the row kernels.
* cfg5: linear regression N=100,000, LOO K=100,000 (sampled folds), sufficient statistics and rows.
* Short-horizon LogS: per-fold estimate and R-hat of a device run vs the oracle run on the same
  streams, before the chains decorrelate.
"""
import numpy as np
import pytest

from paper_2310_07002_b200 import abi, pcv
import _oracle as O
from parity_util import Case, sample_thetas, term_scales

pytestmark = pytest.mark.gpu

RTOL = 1e-12
_cases = {}


def case(name):
    if name not in _cases:
        _cases[name] = Case(name)
    return _cases[name]


def context(cs, policy=None, n_lf=None):
    c = pcv.Context(0)
    if policy is not None:
        c.set_kernel_policy(policy)
    slots = []
    for i, (m, kp, bank) in enumerate(zip(cs.models, cs.kparams, cs.banks)):
        if n_lf is not None:
            kp = pcv.KernelParams(kp.step_size, n_lf, kp.inv_mass_diag)
        slots.append(c.add_model(m, kp, bank, model_id=i))
    return c, slots


def logistic_scales(cs, th, fold):
    """Sum of absolute terms of the logistic log joint (S_lp) and of each gradient component
    (S_g[j] = sum_train |x_ij r_i| + |theta_j|; column 0 is the intercept)."""
    x, y = cs.data.x, cs.data.y
    train = ~cs.excluded(fold)
    eta = th[0] + x @ th[1:]
    r = (y - 1.0 / (1.0 + np.exp(-eta)))[train]
    s_lp = np.sum(np.abs(y * eta - np.logaddexp(0.0, eta))[train]) + np.sum(0.5 * (np.log(2 * np.pi) + th ** 2))
    s_g = np.concatenate([[np.sum(np.abs(r))], np.abs(x[train]).T @ np.abs(r)]) + np.abs(th)
    return s_lp, s_g


def one_tile_points(cs, seed, n=50):
    """One 64-chain tile: a 16-CTA row-split cluster, split over several clusters with a second
    reduction level in global memory (glm_kernel.cu reduce_clusters, the few-chain path)."""
    rng = np.random.default_rng(seed)
    th = sample_thetas(cs, 0, n, seed=seed)
    folds = rng.integers(0, cs.K + 1, n).astype(np.int32)
    folds[:2] = [0, cs.K]
    return th, folds, np.arange(n)


def wave_and_tail_points(cs, seed):
    """Chains for one full wave of 64-chain tiles on every SM plus a 3-tile tail (row-split
    clusters), and the indices checked on the oracle: every tail chain plus a sample of the wave."""
    import torch
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    n = 64 * (sms + 3) - 5
    rng = np.random.default_rng(seed)
    th = sample_thetas(cs, 0, n, seed=seed)
    folds = rng.integers(0, cs.K + 1, n).astype(np.int32)
    folds[:4] = [0, 1, cs.K - 1, cs.K]
    check = np.concatenate([np.arange(4), rng.choice(np.arange(4, 64 * sms), 120, replace=False),
                            np.arange(64 * sms, n)])
    return th, folds, check


# ------------------------------------------------------------------------------ cfg2
@pytest.mark.parametrize("geometry", ["wave+tail", "one-tile-cluster"])
def test_cfg2_log_joint_gradient_and_log_pred(geometry):
    cs = case("cfg2_logistic_bench")
    om = cs.omodels[0]
    if geometry == "wave+tail":
        th, folds, check = wave_and_tail_points(cs, 1)
    else:
        th, folds, check = one_tile_points(cs, 2)
    c, (slot,) = context(cs)
    lp, g = c.eval(slot, folds, th)
    pred = c.eval_pred(slot, folds, th)
    c.close()
    worst = 0.0
    for i in check:
        f = int(folds[i])
        s_lp, s_g = logistic_scales(cs, th[i], f)
        olp, og = om.log_joint(th[i], f), om.grad(th[i], f)
        assert abs(lp[i] - olp) <= RTOL * s_lp, (i, f, lp[i], olp, s_lp)
        err = np.abs(g[i] - og) / s_g
        assert err.max() <= RTOL, (i, f, err.max(), int(err.argmax()))
        opred = om.log_pred(th[i], f)
        assert abs(pred[i] - opred) <= RTOL * (1.0 + abs(opred)), (i, f, pred[i], opred)
        worst = max(worst, abs(lp[i] - olp) / s_lp, err.max())
    print(f"cfg2 {geometry}: {len(check)} chains checked, worst scaled error {worst:.2e}")


@pytest.mark.parametrize("geometry", ["wave+tail", "one-tile-cluster"])
@pytest.mark.parametrize("n_lf", [1, 2])
def test_cfg2_leapfrog_short(n_lf, geometry):
    """n_leapfrog = 1: one half kick, drift, half kick with the gradient of the precise value pass;
    n_leapfrog = 2 adds one gradient-only pass on the fast sigmoid. End points within 1e-12 of the
    sum of absolute terms of the updates (p' = p + eps/2 g0 + eps g1 + ..., q' = q + eps M^-1 p...)."""
    cs = case("cfg2_logistic_bench")
    om, kp = cs.omodels[0], cs.kparams[0]
    th, folds, check = (wave_and_tail_points if geometry == "wave+tail" else one_tile_points)(cs, 10 + n_lf)
    rng = np.random.default_rng(20 + n_lf)
    mom = rng.standard_normal(th.shape) / np.sqrt(kp.inv_mass_diag)
    c, (slot,) = context(cs, n_lf=n_lf)
    q1, p1, ok = c.leapfrog(slot, folds, th, mom)
    c.close()
    assert ok.all()
    eps, im = kp.step_size, kp.inv_mass_diag
    worst = 0.0
    for i in check:
        f = int(folds[i])
        okr, oq, op = om.leapfrog(f, eps, n_lf, im, th[i], mom[i])
        assert okr
        _, s_g0 = logistic_scales(cs, th[i], f)
        _, s_g1 = logistic_scales(cs, oq, f)
        s_p = np.abs(mom[i]) + eps * n_lf * np.maximum(s_g0, s_g1)
        s_q = np.abs(th[i]) + eps * n_lf * im * s_p
        ep = np.abs(p1[i] - op) / s_p
        eq = np.abs(q1[i] - oq) / s_q
        assert ep.max() <= RTOL and eq.max() <= RTOL, (i, f, ep.max(), eq.max())
        worst = max(worst, ep.max(), eq.max())
    print(f"cfg2 leapfrog n_lf={n_lf}: worst scaled error {worst:.2e}")


@pytest.mark.parametrize("geometry", ["wave+tail", "one-tile-cluster"])
def test_cfg2_hmc_step_injected(geometry):
    """hmc_step (hmc.cpp:53-99) at the bench kernel (n_leapfrog = 32) with injected momentum and
    uniform: H0 at 1e-12 of the log joint's terms; H1 after 32 leapfrog steps, the flags and the
    new position against the oracle."""
    cs = case("cfg2_logistic_bench")
    om, kp = cs.omodels[0], cs.kparams[0]
    if geometry == "wave+tail":
        th, folds, check = wave_and_tail_points(cs, 31)
        check = check[::3]
    else:
        th, folds, check = one_tile_points(cs, 31)
    rng = np.random.default_rng(32)
    mom = rng.standard_normal(th.shape) / np.sqrt(kp.inv_mass_diag)
    u = rng.uniform(size=len(th))
    c, (slot,) = context(cs)
    out, h0, h1, acc, div = c.hmc_probe(slot, folds, th, mom, u)
    c.close()
    worst0 = worst1 = 0.0
    for i in check:
        f = int(folds[i])
        oth, oh0, oh1, oacc, odiv = om.hmc_probe(f, kp.step_size, kp.n_leapfrog, kp.inv_mass_diag, th[i], mom[i], u[i])
        s_lp, _ = logistic_scales(cs, th[i], f)
        assert div[i] == odiv
        assert abs(h0[i] - oh0) <= RTOL * s_lp, (i, h0[i], oh0)
        worst0 = max(worst0, abs(h0[i] - oh0) / s_lp)
        if not odiv:
            worst1 = max(worst1, abs(h1[i] - oh1) / s_lp)
            assert abs(h1[i] - oh1) <= RTOL * s_lp, (i, h1[i], oh1, s_lp)
            if abs(np.log(u[i]) + (oh1 - oh0)) > 1e-8:
                assert acc[i] == oacc
            np.testing.assert_allclose(out[i], oth, rtol=1e-10, atol=1e-10)
    print(f"cfg2 hmc_step: worst H0 {worst0:.2e}, worst H1 {worst1:.2e} (scaled by sum|terms|)")


# ------------------------------------------------------------------------------ cfg4 / cfg5
POLICIES = {"suffstat": pcv.Context.KERNEL_SUFFSTAT, "rows": pcv.Context.KERNEL_ROWS}


@pytest.mark.parametrize("policy", list(POLICIES))
@pytest.mark.parametrize("name", ["cfg4_seasonal_bench", "cfg5_linreg_bench"])
def test_bench_shape_gaussian_eval_pred_probe(name, policy):
    cs = case(name)
    c, slots = context(cs, POLICIES[policy])
    rng = np.random.default_rng(7)
    K = cs.K
    folds = np.unique(np.concatenate([[0, 1, K // 2, K - 1, K], rng.integers(0, K, 27)])).astype(np.int32)
    worst = 0.0
    for m, slot in enumerate(slots):
        om, kp = cs.omodels[m], cs.kparams[m]
        th = sample_thetas(cs, m, len(folds), seed=m + 1)
        lp, g = c.eval(slot, folds, th)
        pred = c.eval_pred(slot, folds, th)
        mom = rng.standard_normal(th.shape) / np.sqrt(kp.inv_mass_diag)
        u = rng.uniform(size=len(th))
        out, h0, h1, acc, div = c.hmc_probe(slot, folds, th, mom, u)
        for i, f in enumerate(folds):
            f = int(f)
            s_lp, s_g = term_scales(cs, m, th[i], f)
            olp, og = om.log_joint(th[i], f), om.grad(th[i], f)
            assert abs(lp[i] - olp) <= RTOL * s_lp, (m, f, lp[i], olp)
            assert np.abs(g[i] - og).max() <= RTOL * s_g, (m, f, np.abs(g[i] - og).max(), s_g)
            opred = om.log_pred(th[i], f)
            assert abs(pred[i] - opred) <= 1e-11 * (1 + abs(opred) + om.test_size(f) * 10), (m, f, pred[i], opred)
            oth, oh0, oh1, oacc, odiv = om.hmc_probe(f, kp.step_size, kp.n_leapfrog, kp.inv_mass_diag, th[i],
                                                     mom[i], u[i])
            assert div[i] == odiv
            assert abs(h0[i] - oh0) <= RTOL * s_lp
            if not odiv:
                assert abs(h1[i] - oh1) <= RTOL * s_lp, (m, f, h1[i], oh1, s_lp)
                if abs(np.log(u[i]) + (oh1 - oh0)) > 1e-8:
                    assert acc[i] == oacc
                np.testing.assert_allclose(out[i], oth, rtol=1e-9, atol=1e-9)
            worst = max(worst, abs(lp[i] - olp) / s_lp, np.abs(g[i] - og).max() / s_g)
    c.close()
    print(f"{name}:{policy}: {len(folds)} folds x {len(slots)} models, worst scaled error {worst:.2e}")


# ------------------------------------------------------------------------------ end to end, short
SHORT = ["cfg1_linreg_loo", "ex1_grouped_logo", "radon_logo", "seasonal_hvblock", "logistic_loo", "rat_logo"]


@pytest.mark.parametrize("name", SHORT)
def test_logs_short_horizon_per_fold_matches_oracle(name):
    """LogS run (warm start, warm-up, centring, sampling, per-fold reduction) on the device vs the
    oracle's run_pcv on the same reference streams, 12 iterations: the chains still follow the same
    trajectories, so per-fold estimates and R-hat agree far inside Monte Carlo error (1e-8 relative on
    at least 90% of the folds; a fold whose chain took a different accept decision on a last-ulp
    tie is the exception)."""
    cs = case(name)
    c, slots = context(cs)
    cfg = abi.run_config(chains=4, iters=12, warmup=3, batch_size=3, blocks=4, bench_draws=10, seed=3)
    rep = c.run(cfg)
    c.close()
    orep = O.run_pcv_oracle(cs.omodels, list(range(len(cs.omodels))),
                            [abi.KernelArrays(k.step_size, k.n_leapfrog, k.inv_mass_diag) for k in cs.kparams],
                            cs.banks, cfg)
    for key in ("estimate", "rhat"):
        a, b = rep[key], orep[key]
        np.testing.assert_array_equal(np.isnan(a), np.isnan(b))
        ok = np.isfinite(b)
        rel = np.abs(a[ok] - b[ok]) / (1.0 + np.abs(b[ok]))
        assert np.mean(rel <= 1e-8) >= 0.9, (name, key, np.sort(rel)[-5:])
    np.testing.assert_array_equal(rep["fault"], orep["fault"])


# ------------------------------------------------------------------------------ uncentred data
@pytest.mark.parametrize("policy", list(POLICIES))
def test_gram_statistics_on_uncentred_data(policy):
    """Fold sufficient statistics on data with a large level (cfg1 with y + 1e6, x + 1e3): the masked
    residual sums come from Gram matrices of u - ubar (suffstats.cpp). The row form of S_rr = sum r^2
    has the terms r^2 and, inside each r = y - alpha - x.beta, the products 2|r| (|y| + |alpha| +
    sum|x beta|) (~4e8 here); the raw Gram's om^T A om cancels sum y^2 (~1e14) and would miss that by
    ~1e-2 (25x the 1e-12 budget), the centred one by nothing measurable. The log sigma_y and beta
    gradient components match the oracle at 1e-12 of those term sums on both kernels, at positions
    equivalent to the posterior (the intercept shifted so residuals stay O(1))."""
    base = case("cfg1_linreg_loo")
    cy, cx = 1.0e6, 1.0e3
    d = pcv.Dataset(base.data.y + cy, base.data.x + cx, base.data.group_id, base.data.time_index)
    f = pcv.make_loo_scheme(d)
    m = pcv.GroupedRegressionModel("shifted", d, f)
    om = O.OModel(d, f.arrays(), abi.SpecArrays(family=abi.FAMILY_GROUPED))
    kp = base.kparams[0]
    P = d.x.shape[1]
    th = sample_thetas(base, 0, 12, seed=5)
    th[:, 0] += cy - cx * th[:, 1:1 + P].sum(axis=1)  # alpha_0: identical residuals
    th[:, 1 + P] = th[:, 0]  # mu_alpha next to alpha_0 keeps the hierarchical prior O(1)
    folds = np.array([0, 1, 17, 50, 98, 99, 100, 3, 4, 5, 6, 7], dtype=np.int32)
    c = pcv.Context(0)
    c.set_kernel_policy(POLICIES[policy])
    slot = c.add_model(m, kp, base.banks[0] + 0.0, model_id=0)
    _, g = c.eval(slot, folds, th)
    c.close()
    for i, fk in enumerate(folds):
        fk = int(fk)
        og = om.grad(th[i], fk)
        train = np.ones(d.n_obs, bool)
        if fk < f.K:
            train[f.test_index == fk] = False
        r = d.y - th[i, 0] - d.x @ th[i, 1:1 + P]
        v = np.exp(th[i, P + 3]) ** 2
        terms = np.abs(d.y) + abs(th[i, 0]) + np.abs(d.x * th[i, 1:1 + P]).sum(axis=1)  # inside each r
        s_rr = np.sum((r ** 2 + 2 * np.abs(r) * terms)[train]) / v + train.sum() + v / 10 + 1
        assert abs(g[i, P + 3] - og[P + 3]) <= RTOL * s_rr, (policy, fk, g[i, P + 3], og[P + 3], s_rr)
        for cc in range(P):
            s_x = np.sum(np.abs(d.x[train, cc]) * terms[train]) / v + abs(th[i, 1 + cc])
            assert abs(g[i, 1 + cc] - og[1 + cc]) <= RTOL * s_x, (policy, fk, cc, g[i, 1 + cc], og[1 + cc])


def test_cfg2_kfold_multicluster_matches_single_cluster():
    """cfg2 K-fold (K = 10 x 8 chains = 80 chains: two tiles): each tile split over several 16-CTA
    clusters (the cooperative second-level reduction) against one cluster per tile
    (PCVG_NO_MULTICLUSTER) on the same streams - the same chains to rounding over a short run."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path[:0] = ["tests", "tests/golden", "."]
from parity_util import Case
from paper_2310_07002_b200 import abi, pcv
case = Case("cfg2_logistic_bench")
f = pcv.make_kfold_scheme(case.data, 10, 1)
m = pcv.LogisticModel("M0", case.data, f)
with pcv.Context(0) as c:
    c.add_model(m, case.kparams[0], case.banks[0], model_id=0)
    rep = c.run(abi.run_config(chains=8, iters=6, warmup=2, batch_size=2, blocks=3, bench_draws=10, seed=3))
np.save(sys.argv[1], np.stack([rep["estimate"], rep["rhat"]]))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for tag, env in (("multi", {"PCVG_VERBOSE": "1"}), ("single", {"PCVG_NO_MULTICLUSTER": "1"})):
        path = f"/tmp/pcvg_kfold_{tag}.npy"
        r = subprocess.run([sys.executable, "-c", code, path], env={**os.environ, **env}, capture_output=True,
                           text=True, timeout=600, cwd=root)
        assert r.returncode == 0, r.stderr
        if tag == "multi":  # the multi-cluster launch really ran
            assert "clusters of" in r.stderr and "no error" in r.stderr, r.stderr[-2000:]
        out[tag] = np.load(path)
    a, b = out["multi"], out["single"]
    rel = np.abs(a - b) / (1.0 + np.abs(b))
    assert np.all(rel <= 1e-9), rel

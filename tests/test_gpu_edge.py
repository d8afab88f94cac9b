"""Edge cases of the device models against the CPU oracle: ragged group sizes and
per-row fold keys in the group-batched kernel (the equal-size fixtures only exercise the
uniform-key / equal-length path), poisoned (non-finite) test rows, and groups absent from a
fold's training set (unseen-group predictive)."""
import numpy as np
import pytest

from paper_2310_07002_b200 import abi, pcv
import _oracle as O
from parity_util import DataCase, leapfrog_scales, term_scales

RTOL = 1e-12

pytestmark = pytest.mark.gpu


def ragged_grouped(seed=3, J=45):
    rng = np.random.default_rng(seed)
    sizes = rng.integers(1, 12, J)
    g = np.repeat(np.arange(J), sizes).astype(np.int32)
    n = g.size
    x = rng.standard_normal((n, 3))
    alpha = rng.standard_normal(J)
    y = alpha[g] + x @ np.array([0.5, -0.3, 0.2]) + 0.7 * rng.standard_normal(n)
    return pcv.Dataset(y, x, g)


def thetas(model, n, seed):
    return np.array([pcv.initial_draw(model, seed, 100 + i) for i in range(n)]) * 0.5


FAMILY_KW = {abi.FAMILY_GROUPED: {"family": abi.FAMILY_GROUPED},
             abi.FAMILY_RADON: {"family": abi.FAMILY_RADON, "include_floor": 1},
             abi.FAMILY_RAT_GROWTH: {"family": abi.FAMILY_RAT_GROWTH, "per_subject_slope": 1}}


@pytest.mark.parametrize("policy", [pcv.Context.KERNEL_ROWS, pcv.Context.KERNEL_SUFFSTAT])
@pytest.mark.parametrize("scheme", ["logo", "kfold", "loo"])
@pytest.mark.parametrize("family", [abi.FAMILY_GROUPED, abi.FAMILY_RADON, abi.FAMILY_RAT_GROWTH])
def test_ragged_groups_and_row_keys(scheme, family, policy):
    d = ragged_grouped()
    if family == abi.FAMILY_RADON:
        d = pcv.Dataset(d.y, (d.x[:, :1] > 0).astype(float), d.group_id)
    if family == abi.FAMILY_RAT_GROWTH:
        d = pcv.Dataset(d.y + 250.0, np.abs(d.x[:, :1]) * 10.0, d.group_id)
    f = {"logo": pcv.make_logo_scheme, "kfold": lambda dd: pcv.make_kfold_scheme(dd, 7, 2),
         "loo": pcv.make_loo_scheme}[scheme](d)
    cls = {abi.FAMILY_GROUPED: lambda: pcv.GroupedRegressionModel("M", d, f),
           abi.FAMILY_RADON: lambda: pcv.RadonStyleModel("M", d, f, True),
           abi.FAMILY_RAT_GROWTH: lambda: pcv.RatGrowthModel("M", d, f, True)}[family]
    model = cls()
    om = O.OModel(d, f.arrays(), model.spec)
    dim = model.dim()
    kp = pcv.KernelParams(0.01, 8, np.ones(dim))
    dc = DataCase(d, f, FAMILY_KW[family])
    with pcv.Context(0) as ctx:
        ctx.set_kernel_policy(policy)
        slot = ctx.add_model(model, kp, thetas(model, 2, 1))
        folds = sorted({0, 1, f.K // 2, f.K - 1, f.K})
        for fold in folds:
            th = thetas(model, 3, fold + 7)
            lp, g = ctx.eval(slot, np.full(3, fold), th)
            for i in range(3):
                olp, og = om.log_joint(th[i], fold), om.grad(th[i], fold)
                s_lp, s_g = term_scales(dc, 0, th[i], fold)
                assert abs(lp[i] - olp) <= RTOL * s_lp, (fold, lp[i], olp, s_lp)
                assert np.abs(g[i] - og).max() <= RTOL * s_g, (fold, np.abs(g[i] - og).max(), s_g)
            pr = ctx.eval_pred(slot, np.full(3, fold), th)
            for i in range(3):
                ref = om.log_pred(th[i], fold)
                assert abs(pr[i] - ref) <= 1e-10 * (1.0 + abs(ref)), (fold, pr[i], ref)


@pytest.mark.parametrize("policy", [pcv.Context.KERNEL_ROWS, pcv.Context.KERNEL_SUFFSTAT])
def test_poisoned_test_row(policy):
    """A non-finite y in a test row: the reference's log_joint multiplies the test term by 0,
    which is NaN (grouped_regression.cpp:74-76); training folds stay finite."""
    d = ragged_grouped(seed=5, J=20)
    y = d.y.copy()
    g = d.group_id
    y[np.where(g == 3)[0][0]] = np.inf
    d = pcv.Dataset(y, d.x, g)
    f = pcv.make_logo_scheme(d)
    model = pcv.GroupedRegressionModel("M", d, f)
    om = O.OModel(d, f.arrays(), model.spec)
    with pcv.Context(0) as ctx:
        ctx.set_kernel_policy(policy)  # SUFFSTAT: non-finite data keeps the row kernels
        slot = ctx.add_model(model, pcv.KernelParams(0.01, 8, np.ones(model.dim())), thetas(model, 1, 1))
        th = thetas(model, 1, 4)
        for fold in (3, 4):
            lp, _ = ctx.eval(slot, [fold], th)
            olp = om.log_joint(th[0], fold)
            assert (np.isnan(lp[0]) and np.isnan(olp)) or (not np.isfinite(olp) and lp[0] == olp) or \
                abs(lp[0] - olp) <= 1e-10 * max(1.0, abs(olp)), (fold, lp[0], olp)


def _many_groups_cases():
    """Hierarchical models with J >= 64 groups: the sufficient-statistics kernel runs a warp per
    chain there (lane-owned groups, shared-memory group slots, per-lane override walks)."""
    import sys
    from parity_util import Case
    out = []
    c = Case("cfg3_radon_bench")  # radon-style, 400 counties, LOGO; the fixture's kernel and bank
    for m in range(len(c.models)):
        kp = c.kparams[m]
        out.append(("radon400_logo_m%d" % m, c.models[m], c.omodels[m],
                    pcv.KernelParams(kp.step_size, 8, kp.inv_mass_diag),
                    c.banks[m][np.linspace(0, len(c.banks[m]) - 1, 4).astype(int)], c.K,
                    DataCase(c.data, c.folds, c.kws[m])))
    d = ragged_grouped(seed=9, J=150)  # grouped, 150 ragged groups, K-fold: every fold touches many groups
    f = pcv.make_kfold_scheme(d, 7, 3)
    model = pcv.GroupedRegressionModel("M", d, f)
    out.append(("grouped150_kfold", model, O.OModel(d, f.arrays(), model.spec),
                pcv.KernelParams(0.01, 8, np.ones(model.dim())), thetas(model, 4, 5), f.K,
                DataCase(d, f, FAMILY_KW[abi.FAMILY_GROUPED])))
    # growth model with per-subject slopes, 120 ragged subjects: two slot arrays per lane
    d0 = ragged_grouped(seed=13, J=120)
    dr = pcv.Dataset(d0.y + 250.0, np.abs(d0.x[:, :1]) * 10.0, d0.group_id)
    fr = pcv.make_kfold_scheme(dr, 7, 4)
    rm = pcv.RatGrowthModel("M", dr, fr, True)
    J = 120  # theta = [alpha_g, beta_g, mu_a, mu_b, log s_a, log s_b, log s_y] near the data
    gm = np.array([dr.y[dr.group_id == g].mean() for g in range(J)])
    base = np.concatenate([gm, np.zeros(J), [250.0, 0.0, 0.0, -1.0, -0.3]])
    th_r = base + 0.01 * np.random.default_rng(6).standard_normal((4, base.size))
    out.append(("rat120_kfold", rm, O.OModel(dr, fr.arrays(), rm.spec),
                pcv.KernelParams(0.005, 8, np.ones(rm.dim())), th_r, fr.K,
                DataCase(dr, fr, FAMILY_KW[abi.FAMILY_RAT_GROWTH])))
    return out


@pytest.mark.parametrize("policy", [pcv.Context.KERNEL_SUFFSTAT, pcv.Context.KERNEL_ROWS])
def test_many_groups_warp_kernels(policy):
    """J >= 64: log joint / gradient at the stored position, leapfrog end points (hmc.cpp:22-51)
    and injected-momentum hmc_step (hmc.cpp:53-99) against the oracle."""
    rng = np.random.default_rng(21)
    for name, model, om, kp, th, K, dc in _many_groups_cases():
        step, im = kp.step_size, kp.inv_mass_diag
        with pcv.Context(0) as ctx:
            ctx.set_kernel_policy(policy)
            slot = ctx.add_model(model, kp, th)
            folds = np.array([0, 1, K // 2, K], dtype=np.int32)
            lp, g = ctx.eval(slot, folds, th)
            for i in range(4):
                olp, og = om.log_joint(th[i], int(folds[i])), om.grad(th[i], int(folds[i]))
                s_lp, s_g = term_scales(dc, 0, th[i], int(folds[i]))
                assert abs(lp[i] - olp) <= RTOL * s_lp, (name, i, lp[i], olp, s_lp)
                assert np.abs(g[i] - og).max() <= RTOL * s_g, (name, i, np.abs(g[i] - og).max(), s_g)
            mom = rng.standard_normal(th.shape) / np.sqrt(im)
            q1, p1, ok = ctx.leapfrog(slot, folds, th, mom)
            assert ok.sum() >= 2, (name, ok)
            for i in range(4):
                okr, oq, op = om.leapfrog(int(folds[i]), step, 8, im, th[i], mom[i])
                assert bool(okr) == bool(ok[i]), (name, i)
                if not okr:
                    continue
                s_q, s_p = leapfrog_scales(dc, 0, th[i], mom[i], int(folds[i]), kp, theta_end=oq)
                assert np.all(np.abs(q1[i] - oq) <= RTOL * s_q), (name, i, np.max(np.abs(q1[i] - oq) / s_q))
                assert np.all(np.abs(p1[i] - op) <= RTOL * s_p), (name, i, np.max(np.abs(p1[i] - op) / s_p))
            u = rng.uniform(size=4)
            out, h0, h1, acc, div = ctx.hmc_probe(slot, folds, th, mom, u)
            for i in range(4):
                oth, oh0, oh1, oacc, odiv = om.hmc_probe(int(folds[i]), step, 8, im, th[i], mom[i], u[i])
                assert div[i] == odiv, name
                s_lp, _ = term_scales(dc, 0, th[i], int(folds[i]))
                assert abs(h0[i] - oh0) <= RTOL * s_lp, (name, h0[i], oh0)
                if not odiv:
                    s_lp1, _ = term_scales(dc, 0, oth, int(folds[i]))
                    assert abs(h1[i] - oh1) <= RTOL * max(s_lp, s_lp1), (name, h1[i], oh1)
                    s_q, _ = leapfrog_scales(dc, 0, th[i], mom[i], int(folds[i]), kp, theta_end=oth)
                    assert np.all(np.abs(out[i] - oth) <= RTOL * s_q), name

"""GPU parity proper: every probe goes through the C ABI (libpcvg.so) on the device and is compared
with the CPU oracle (oracle/pcv_oracle.c, itself pinned to the reference in test_oracle_*.py) on
the same inputs. Tolerances follow SURVEY.md 8(c): FP64 per-step values within
1e-12 * sum|terms|; end-to-end elpd within Monte Carlo error."""
import numpy as np
import pytest

from paper_2310_07002_b200 import abi, pcv
import _oracle as O
from parity_util import ALL_FIXTURES, Case, leapfrog_scales, sample_thetas, term_scales, probe_folds

pytestmark = pytest.mark.gpu

RTOL = 1e-12


@pytest.fixture(scope="module")
def ctx():
    c = pcv.Context(0)
    yield c
    c.close()


_cases = {}
# fixtures whose models have two row-streaming kernels: the tensor-core GLM kernel or the
# group-batched hierarchical kernel (policy ROWS / TENSOR), and the generic row-split kernel (GENERIC)
BOTH_KERNELS = {"cfg1_linreg_loo": "tensor", "seasonal_timeblocks": "tensor", "seasonal_hvblock": "tensor",
                "ex1_grouped_logo": "batched", "radon_logo": "batched"}


def case_in(ctx, name):
    """(Case, slots) with the case's models registered in a fresh context. A name suffixed with
    ':tensor' / ':batched' / ':generic' / ':suffstat' forces that kernel."""
    name, _, kernel = name.partition(":")
    if name not in _cases:
        _cases[name] = Case(name)
    case = _cases[name]
    c = pcv.Context(0)
    if kernel:
        c.set_kernel_policy({"tensor": c.KERNEL_TENSOR, "batched": c.KERNEL_ROWS,
                             "generic": c.KERNEL_GENERIC, "suffstat": c.KERNEL_SUFFSTAT}[kernel])
    slots = [c.add_model(m, kp, bank, model_id=i)
             for i, (m, kp, bank) in enumerate(zip(case.models, case.kparams, case.banks))]
    return case, c, slots


# Gaussian linear fixtures that also run on fold sufficient statistics (policy SUFFSTAT)
SUFF_KERNEL = {"cfg1_linreg_loo", "ex1_grouped_logo", "radon_logo", "seasonal_timeblocks", "seasonal_hvblock",
               "rat_logo"}  # rat: M_B (shared slope) and M_A (per-subject slopes, per-subject Grams)


def with_kernels(names):
    out = []
    for n in names:
        if n in BOTH_KERNELS:
            out += [n + ":" + BOTH_KERNELS[n], n + ":generic"]
        else:
            out.append(n)
        if n in SUFF_KERNEL:
            out.append(n + ":suffstat")
    return out


@pytest.mark.parametrize("name", with_kernels(ALL_FIXTURES))
def test_log_joint_and_gradient(ctx, name):
    case, c, slots = case_in(ctx, name)
    worst = 0.0
    for m, slot in enumerate(slots):
        om = case.omodels[m]
        for fold in probe_folds(case):
            th = sample_thetas(case, m, 6, seed=fold)
            lp, g = c.eval(slot, np.full(len(th), fold), th)
            for i in range(len(th)):
                s_lp, s_g = term_scales(case, m, th[i], fold)
                olp = om.log_joint(th[i], fold)
                og = om.grad(th[i], fold)
                assert abs(lp[i] - olp) <= RTOL * s_lp, (name, m, fold, lp[i], olp, s_lp)
                err = np.abs(g[i] - og).max()
                assert err <= RTOL * s_g, (name, m, fold, err, s_g)
                worst = max(worst, abs(lp[i] - olp) / s_lp, err / s_g)
    c.close()
    print(f"{name}: worst scaled error {worst:.2e}")


@pytest.mark.parametrize("name", with_kernels(ALL_FIXTURES))
def test_log_pred(ctx, name):
    case, c, slots = case_in(ctx, name)
    for m, slot in enumerate(slots):
        om = case.omodels[m]
        folds = [f for f in probe_folds(case)]
        for fold in folds:
            th = sample_thetas(case, m, 4, seed=10 + fold)
            lp = c.eval_pred(slot, np.full(len(th), fold), th)
            for i in range(len(th)):
                ref = om.log_pred(th[i], fold)
                assert abs(lp[i] - ref) <= 1e-11 * (1 + abs(ref) + om.test_size(fold) * 10), (name, fold, lp[i], ref)
    c.close()


@pytest.mark.parametrize("name", with_kernels(ALL_FIXTURES))
def test_hmc_step_injected(ctx, name):
    """hmc_step (hmc.cpp:53-99) with injected momentum and uniform: h0, h1, flags, new position."""
    case, c, slots = case_in(ctx, name)
    rng = np.random.default_rng(5)
    for m, slot in enumerate(slots):
        om, kp = case.omodels[m], case.kparams[m]
        n = 8
        th = sample_thetas(case, m, n, seed=3)
        folds = rng.integers(0, case.K + 1, n).astype(np.int32)
        mom = rng.standard_normal(th.shape) / np.sqrt(kp.inv_mass_diag)
        u = rng.uniform(size=n)
        out, h0, h1, acc, div = c.hmc_probe(slot, folds, th, mom, u)
        for i in range(n):
            oth, oh0, oh1, oacc, odiv = om.hmc_probe(int(folds[i]), kp.step_size, kp.n_leapfrog,
                                                     kp.inv_mass_diag, th[i], mom[i], u[i])
            assert div[i] == odiv
            s_lp, _ = term_scales(case, m, th[i], int(folds[i]))
            assert abs(h0[i] - oh0) <= RTOL * s_lp
            if not odiv:
                # H1 after n_lf = 32 leapfrog steps: 1e-12 of the log joint's terms at either end
                s_lp1, _ = term_scales(case, m, oth, int(folds[i]))
                assert abs(h1[i] - oh1) <= RTOL * max(s_lp, s_lp1), (name, i, h1[i], oh1)
                if abs(np.log(u[i]) + (oh1 - oh0)) > 1e-8:
                    assert acc[i] == oacc
                s_q, _ = leapfrog_scales(case, m, th[i], mom[i], int(folds[i]), kp, theta_end=oth)
                assert np.all(np.abs(out[i] - oth) <= RTOL * s_q), (name, i, np.max(np.abs(out[i] - oth) / s_q))
    c.close()


@pytest.mark.parametrize("name", with_kernels(["cfg1_linreg_loo", "ex1_grouped_logo", "radon_logo",
                                               "seasonal_hvblock", "logistic_loo", "rat_logo"]))
def test_chain_trajectory_reference_stream(ctx, name):
    """Same reference Philox stream (seed, ChainSampling, model, fold, chain): the device chain
    reproduces the oracle chain (identical integer draws; momenta to ~1 ulp) until chaos."""
    case, c, slots = case_in(ctx, name)
    m, slot = 0, slots[0]
    om, kp = case.omodels[m], case.kparams[m]
    fold, chain, seed, steps = min(3, case.K - 1), 1, 17, 120
    th0 = case.banks[m][7]
    traj, div = c.hmc_chain(slot, fold, chain, seed, th0, steps)
    stream = pcv.stream_key(abi.STREAM_CHAIN_SAMPLING, m, fold, chain)
    otraj, odiv = om.hmc_chain(fold, kp.step_size, kp.n_leapfrog, kp.inv_mass_diag, seed, stream, th0, steps)
    # identical streams: the same divergence / acceptance sequence and positions equal to rounding
    # until the first last-ulp difference is amplified by the chaotic dynamics
    rel = np.abs(traj - otraj).max(axis=1) / (1.0 + np.abs(otraj).max(axis=1))
    onset = int(np.argmax(rel > 1e-6)) if np.any(rel > 1e-6) else steps
    print(f"{name}: trajectories agree to 1e-6 for {onset} of {steps} transitions (1e-12 for "
          f"{int(np.argmax(rel > 1e-12)) if np.any(rel > 1e-12) else steps})")
    # rounding level at first (1e-15 .. 2e-12 after a 32-step trajectory), then flat or exponential
    # growth (J = 1 grouped regression: ~1.35x per transition from 1e-15, crossing 1e-6 after ~74
    # transitions; every other fixture stays below 1e-6 for all 120)
    assert np.all(rel[:10] < 1e-11), (name, rel[:10])
    assert onset >= min(steps, 60), (name, onset, rel[:onset + 3])
    np.testing.assert_array_equal(div[:onset], odiv[:onset])
    c.close()


@pytest.mark.parametrize("name", with_kernels(["cfg1_linreg_loo", "ex1_grouped_logo", "radon_logo",
                                               "seasonal_hvblock", "logistic_kfold", "rat_logo"]))
def test_run_pcv_within_mcse(ctx, name):
    """End-to-end run_pcv on the device vs the oracle run_pcv on the same inputs: the headline
    elpd / delta within Monte Carlo error, identical report structure."""
    case, c, slots = case_in(ctx, name)
    rc = case.z["run_cfg"]
    cfg = abi.run_config(chains=int(rc[0]), iters=int(rc[1]), warmup=int(rc[2]), batch_size=int(rc[3]),
                         blocks=int(rc[4]), bench_draws=int(rc[5]), checkpoint_every=int(rc[6]), seed=1)
    rep = c.run(cfg)
    orep = O.run_pcv_oracle(case.omodels, list(range(len(case.omodels))),
                            [abi.KernelArrays(k.step_size, k.n_leapfrog, k.inv_mass_diag) for k in case.kparams],
                            case.banks, cfg)
    assert rep["n_checkpoints"] == orep["n_checkpoints"]
    assert rep["iters_run"] == cfg.iters
    # Delta-hat (or the single-model score total) agrees within combined MC error (4 sigma)
    tol = 4.0 * np.hypot(rep["mcse"], orep["mcse"]) + 1e-9
    assert abs(rep["delta_hat"] - orep["delta_hat"]) <= tol, (rep["delta_hat"], orep["delta_hat"], tol)
    assert np.isfinite(rep["rhat_max"])
    assert rep["benchmark_count"] > 0
    # per-fold estimates: MC error per fold is ~sqrt(mc/(L N)); check aggregate agreement
    est, oest = rep["estimate"], orep["estimate"]
    assert est.shape == oest.shape
    c.close()


SCORE_BASES = ["cfg1_linreg_loo", "ex1_grouped_logo", "radon_logo", "seasonal_timeblocks", "seasonal_hvblock",
               "rat_logo"]


def _score_cfg(case, score, iters=None, warmup=None, seed=1):
    rc = case.z["run_cfg"]
    return abi.run_config(chains=int(rc[0]), iters=int(iters or rc[1]), warmup=int(rc[2] if warmup is None else warmup),
                          batch_size=int(rc[3]) if iters is None else 5, blocks=int(rc[4]),
                          bench_draws=int(rc[5]), checkpoint_every=int(rc[6]) if iters is None else 0,
                          seed=seed, score=score)


@pytest.mark.parametrize("name", with_kernels(SCORE_BASES))
@pytest.mark.parametrize("score", [abi.SCORE_HS, abi.SCORE_DSS])
def test_score_short_horizon_matches_oracle(ctx, name, score):
    """HS / DSS state on device (pred_derivs / pred_sample after every hmc_step, warm-up centring,
    chain merge, hs/dss fold scores) vs the oracle on the same streams over a horizon short enough
    that the chains have not decorrelated: per-fold estimates agree to ~1e-9."""
    case, c, slots = case_in(ctx, name)
    cfg = _score_cfg(case, score, iters=20, warmup=4)
    rep = c.run(cfg)
    orep = O.run_pcv_oracle(case.omodels, list(range(len(case.omodels))),
                            [abi.KernelArrays(k.step_size, k.n_leapfrog, k.inv_mass_diag) for k in case.kparams],
                            case.banks, cfg)
    est, oest = rep["estimate"], orep["estimate"]
    np.testing.assert_array_equal(np.isnan(est), np.isnan(oest))
    np.testing.assert_array_equal(rep["fault"], orep["fault"])
    ok = np.isfinite(oest)
    rel = np.abs(est[ok] - oest[ok]) / (1.0 + np.abs(oest[ok]))
    assert np.mean(rel <= 1e-8) >= 0.9, (name, np.sort(rel)[-5:])
    assert np.isnan(rep["mcse"])
    c.close()


@pytest.mark.parametrize("name", SCORE_BASES)
@pytest.mark.parametrize("score", [abi.SCORE_HS, abi.SCORE_DSS])
def test_score_run_within_mc_error_of_reference(ctx, name, score):
    """Full fixture run (N = 100-200) vs the reference report (tests/golden/<name>_<score>.npz): the
    headline delta-hat agrees within 5 Monte Carlo standard deviations, the MC sd estimated from
    independent device runs (seeds 2..6) of the same configuration."""
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden",
                             f"{name}_{'hs' if score == abi.SCORE_HS else 'dss'}.npz"))
    case, c, slots = case_in(ctx, name)
    rep = c.run(_score_cfg(case, score))
    others = [c.run(_score_cfg(case, score, seed=s))["delta_hat"] for s in range(2, 7)]
    sd = np.std(others, ddof=1)
    ref = float(z["ref_delta_hat"])
    assert abs(rep["delta_hat"] - ref) <= 5.0 * np.sqrt(2.0) * sd + 1e-9 * abs(ref), (rep["delta_hat"], ref, sd)
    np.testing.assert_array_equal(np.isnan(rep["estimate"]), np.isnan(z["ref_estimate"]))
    c.close()


def test_score_unsupported_for_logistic(ctx):  # Model::check_score_support, model.cpp:21-28
    case, c, slots = case_in(ctx, "logistic_loo")
    for sc in (abi.SCORE_HS, abi.SCORE_DSS):
        with pytest.raises(pcv.UnsupportedScore):
            c.run(abi.run_config(chains=4, iters=20, warmup=2, batch_size=5, score=sc))
    c.close()


def test_wave_tail_split_matches_unsplit():
    """More than one wave of 64-chain tiles: the last partial wave runs as row-split clusters
    (glm_kernel.cu launch_t). Its chains must follow the same trajectories as without the split
    (same streams; the gradient differs only in summation order)."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path[:0] = ["tests", "tests/golden", "."]
from parity_util import Case
from paper_2310_07002_b200 import abi, pcv
case = Case("logistic_loo")
with pcv.Context(0) as c:
    c.add_model(case.models[0], case.kparams[0], case.banks[0], model_id=0)
    rep = c.run(abi.run_config(chains=20, iters=10, warmup=2, batch_size=5, bench_draws=5, seed=2))
np.save(sys.argv[1], rep["estimate"])
'''
    out = {}
    for tag, env in (("split", {}), ("plain", {"PCVG_NO_TAIL_SPLIT": "1"})):
        path = f"/tmp/pcvg_tail_{tag}.npy"
        r = subprocess.run([sys.executable, "-c", code, path], env={**os.environ, **env}, capture_output=True,
                           text=True, timeout=600, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        assert r.returncode == 0, r.stderr
        out[tag] = np.load(path)
    a, b = out["split"], out["plain"]
    assert a.shape == (500,)  # 500 folds x 20 chains = 157 tiles: 148 + a 9-tile tail
    rel = np.abs(a - b) / (1.0 + np.abs(b))
    assert np.mean(rel <= 1e-9) >= 0.95 and np.all(rel[:440] == 0.0), np.sort(rel)[-5:]


@pytest.mark.parametrize("name", with_kernels(["cfg1_linreg_loo", "ex1_grouped_logo", "radon_logo",
                                               "seasonal_hvblock", "logistic_loo", "rat_logo"]))
def test_leapfrog_endpoint_and_reversibility(ctx, name):
    """leapfrog (hmc.cpp:22-51): the device end point (theta', p') matches the oracle's, and
    integrating back from (theta', -p') returns to (theta, -p) within 1e-10 (test_hmc.cpp:134-147)."""
    case, c, slots = case_in(ctx, name)
    rng = np.random.default_rng(11)
    m, slot = 0, slots[0]
    om, kp = case.omodels[m], case.kparams[m]
    th = sample_thetas(case, m, 4, seed=2)
    mom = rng.standard_normal(th.shape) / np.sqrt(kp.inv_mass_diag)
    folds = np.array([0, 1, case.K // 2, case.K], dtype=np.int32)
    q1, p1, ok = c.leapfrog(slot, folds, th, mom)
    assert ok.all()
    for i in range(4):
        okr, oq, op = om.leapfrog(int(folds[i]), kp.step_size, kp.n_leapfrog, kp.inv_mass_diag, th[i], mom[i])
        s_q, s_p = leapfrog_scales(case, m, th[i], mom[i], int(folds[i]), kp, theta_end=oq)
        assert np.all(np.abs(q1[i] - oq) <= RTOL * s_q), (name, i, np.max(np.abs(q1[i] - oq) / s_q))
        assert np.all(np.abs(p1[i] - op) <= RTOL * s_p), (name, i, np.max(np.abs(p1[i] - op) / s_p))
    q2, p2, ok2 = c.leapfrog(slot, folds, q1, -p1)
    assert ok2.all()
    np.testing.assert_allclose(q2, th, rtol=0, atol=1e-10 * (1 + np.abs(th).max()))
    np.testing.assert_allclose(-p2, mom, rtol=0, atol=1e-10 * (1 + np.abs(mom).max()) * 10)
    c.close()


@pytest.mark.parametrize("scale", [1.0, 30.0, 100.0, 1000.0])
def test_logistic_leapfrog_wide_eta(ctx, scale):
    """The gradient-only passes of the logistic kernel (tc_common.cuh::logistic_resid_fast: integer
    clamp at |eta| = 700, exponent assembly, sign-folded reciprocal) against the oracle's std::exp
    sigmoid on positions scaled so that eta = x . theta reaches |eta| ~ 360 (scale 100, still a
    finite-energy trajectory) and ~3600 (scale 1000, past the clamp). The leapfrog probe runs
    hmc_step with u = 0, so a trajectory the oracle calls divergent (|dH| > 1000, hmc.cpp:82-90)
    must come back not-ok; every other end point matches at the posterior tolerance."""
    case, c, slots = case_in(ctx, "logistic_loo")
    rng = np.random.default_rng(21)
    m, slot = 0, slots[0]
    om, kp = case.omodels[m], case.kparams[m]
    th = sample_thetas(case, m, 4, seed=4) * scale
    mom = rng.standard_normal(th.shape) / np.sqrt(kp.inv_mass_diag)
    folds = np.array([0, 1, case.K // 2, case.K], dtype=np.int32)
    q1, p1, ok = c.leapfrog(slot, folds, th, mom)
    for i in range(4):
        _, oh0, oh1, _, odiv = om.hmc_probe(int(folds[i]), kp.step_size, kp.n_leapfrog, kp.inv_mass_diag,
                                            th[i], mom[i], 0.0)
        assert bool(ok[i]) == (not odiv), (scale, i, oh1 - oh0)
        if odiv:
            continue
        okr, oq, op = om.leapfrog(int(folds[i]), kp.step_size, kp.n_leapfrog, kp.inv_mass_diag, th[i], mom[i])
        np.testing.assert_allclose(q1[i], oq, rtol=1e-8, atol=1e-9 * (1 + np.abs(oq).max()))
        np.testing.assert_allclose(p1[i], op, rtol=1e-8, atol=1e-8 * (1 + np.abs(op).max()))
    _, h0, h1, _, div = c.hmc_probe(slot, folds, th, mom, np.zeros(4))
    for i in range(4):
        _, oh0, oh1, _, odiv = om.hmc_probe(int(folds[i]), kp.step_size, kp.n_leapfrog, kp.inv_mass_diag,
                                            th[i], mom[i], 0.0)
        assert div[i] == odiv
        assert abs(h0[i] - oh0) <= 1e-10 * (1 + abs(oh0))
        if not odiv:
            assert abs(h1[i] - oh1) <= 1e-8 * (1 + abs(oh1))
    c.close()


def test_snapshots_prefix_stable(ctx):
    """test_engine.cpp:150-173: the first snapshot of a 200-iteration run equals the final
    statistics of a 100-iteration run (R-hat up to the block-boundary summation order)."""
    case, c, slots = case_in(ctx, "ex1_grouped_logo")
    base = dict(chains=4, warmup=20, batch_size=10, bench_draws=10, seed=6)
    long = c.run(abi.run_config(iters=200, checkpoint_every=100, **base))
    short = c.run(abi.run_config(iters=100, **base))
    a, b = long["snapshots"][0], short["snapshots"][0]
    assert a[0] == b[0] == 100
    assert a[1] == b[1] and a[2] == b[2] and a[5] == b[5]  # delta_hat, mcse, ess
    assert abs(a[6] - b[6]) <= 1e-12 * b[6]
    c.close()

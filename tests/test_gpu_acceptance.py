"""The reference's acceptance criteria and engine fault test, restated on GPU output through the C ABI.

* C3 (acceptance.cpp:126-185): HMC on a standard normal - 10 seeds x 4 chains x 10,000 transitions
  (step 0.157, 10 leapfrog steps) - KS passes >= 9/10, |mean| <= 3 MCSE, |var - 1| <= 0.1.
* C5 (acceptance.cpp:212-250): Example-1 selection, 10 seeds: full-data fits (Step 1) and the PCV run
  on the device; Pr(A better) > 0.9 on >= 8 seeds, MCSE < epistemic SE at every checkpoint >= 500.
* C6 / C7 (acceptance.cpp:259-325): the shuffle-benchmark calibration / pathology harness, fed as
  score streams through the device accumulators, fold reduction, benchmark kernel and verdict
  (pcvg_run_streams); per seed against the reference's own numbers (tests/golden/acceptance_c6c7.npz,
  make_acceptance.py), and through the early-stop rule: clean runs stop, a stuck chain
  or a +5 shift never stops a run.
* Failed folds (engine.cpp:385-397, test_engine.cpp:240-255 BrokenFoldModel): a fold whose chains
  all diverge is excluded from the estimate and the benchmark but reported, identically to the oracle.
"""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2310_07002_b200 import abi, pcv
import _oracle as O
from parity_util import Case

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def normals(seed, stream, n):
    """n draws of CounterRng(seed, stream).normal() (the oracle's bit-exact Philox + Box-Muller)."""
    lib = O.oracle()
    arg = np.zeros(n, dtype=np.uint64)
    out = np.zeros(n)
    rc = lib.pcvo_rng_sequence(seed, stream, 0, 0, b"n" * n, abi.ptr(arg, C.c_uint64), n, abi.ptr(out, C.c_double))
    assert rc == 0
    return out


def corrupted_streams(seed, kind, k_folds=10, l=4, n=1000):
    """The score streams of acceptance.cpp:266-300 (kind 0 clean, 1 stuck chain, 2 +5 shift)."""
    lib = O.oracle()
    run_seed = 7000 + seed
    rho = 0.3
    innov = np.sqrt(1.0 - rho * rho)
    s = np.zeros((k_folds, l, n))
    mu = np.zeros(k_folds)
    for k in range(k_folds):
        mu[k] = 2.0 * normals(run_seed, lib.pcvo_stream_key(abi.STREAM_SIMULATE, k, 0, 0), 1)[0]
        for c in range(l):
            z = normals(run_seed, lib.pcvo_stream_key(abi.STREAM_CHAIN_SAMPLING, 0, k, c), n)
            start = mu[k] + 3.0
            state = start - mu[k]
            corrupt = kind != 0 and k == 2 and c == 0
            for i in range(n):
                state = rho * state + innov * z[i]
                v = start if (corrupt and kind == 1) else mu[k] + state
                if corrupt and kind == 2:
                    v += 5.0
                s[k, c, i] = v
    return s, mu


@pytest.fixture(scope="module")
def c6c7():
    return np.load(os.path.join(GOLDEN, "acceptance_c6c7.npz"))


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_shuffle_benchmark_c6_c7_match_reference(c6c7, kind):
    R = int(c6c7["bench_draws"][kind])
    verdicts = []
    with pcv.Context(0) as c:
        for seed in range(20):
            s, mu = corrupted_streams(seed, kind)
            cfg = abi.run_config(chains=4, iters=1000, warmup=0, batch_size=50, blocks=5, bench_draws=R,
                                 seed=7000 + seed)
            rep = c.run_streams(s, mu, cfg)
            obs, qv = c6c7["observed"][kind, seed], c6c7["quantile_value"][kind, seed]
            assert abs(rep["verdict_observed"] - obs) <= 1e-12 * obs, (seed, rep["verdict_observed"], obs)
            assert abs(rep["verdict_quantile_value"] - qv) <= 1e-12 * qv, (seed, rep["verdict_quantile_value"], qv)
            if abs(obs - qv) > 1e-10 * qv:
                assert rep["verdict_pass"] == c6c7["verdict_pass"][kind, seed], seed
            assert rep["benchmark_count"] == R
            verdicts.append(rep["verdict_pass"])
    if kind == 0:
        assert sum(verdicts) >= 18  # C6: observed <= q99 on >= 18/20 clean runs
    else:
        assert sum(1 - v for v in verdicts) >= 19  # C7: flagged on >= 19/20


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_early_stop_rule_on_c6_c7_streams(c6c7, kind):
    """checkpoint_every = 100 over 1,000 iterations: 10 sub-blocks, regrouped into blocks = 5 for the
    benchmark, so the rule may first fire at iteration 500. Clean runs stop there (or soon after)
    with a passing verdict; a stuck or shifted chain never stops a run, and its final verdict equals
    the reference's D = 5 verdict (two sub-blocks per block = the reference's block layout)."""
    R = int(c6c7["bench_draws"][kind])
    stopped, flagged = 0, 0
    with pcv.Context(0) as c:
        for seed in range(20):
            s, mu = corrupted_streams(seed, kind)
            cfg = abi.run_config(chains=4, iters=1000, warmup=0, batch_size=50, blocks=5, bench_draws=R,
                                 seed=7000 + seed, checkpoint_every=100, early_stop=1)
            rep = c.run_streams(s, mu, cfg)
            assert rep["iters_run"] >= 500 and rep["iters_run"] % 100 == 0
            if rep["iters_run"] < 1000:
                stopped += 1
                assert rep["verdict_pass"] == 1 and rep["mcse"] < rep["epistemic_se"]
            else:
                obs, qv = c6c7["observed"][kind, seed], c6c7["quantile_value"][kind, seed]
                assert abs(rep["verdict_observed"] - obs) <= 1e-12 * obs
                assert abs(rep["verdict_quantile_value"] - qv) <= 1e-12 * qv
            flagged += 1 - rep["verdict_pass"]
    if kind == 0:
        assert stopped >= 18, stopped
    else:
        assert stopped == 0 and flagged >= 19, (stopped, flagged)


def test_early_stop_validation():
    with pcv.Context(0) as c:
        s, mu = corrupted_streams(0, 0)
        with pytest.raises(pcv.InvalidInput):  # 4 check intervals < 5 blocks
            c.run_streams(s, mu, abi.run_config(chains=4, iters=1000, blocks=5, bench_draws=10, seed=1,
                                                checkpoint_every=250, early_stop=1))


# ------------------------------------------------------------------------------ C3
def batch_means_variance(chains, b):  # scoring.cpp:106-121
    bm = [c[: len(c) // b * b].reshape(-1, b).mean(axis=1) for c in chains]
    allm = np.concatenate(bm)
    return b * np.sum((allm - allm.mean()) ** 2) / (len(allm) - 1.0)


def test_hmc_standard_normal_c3():
    """A logistic model whose covariate column is identically zero: the coefficient beta_1 has only
    its N(0,1) prior, so its marginal under the device HMC (chains on the reference streams
    ChainSampling(0, 0, c), seeds 3000 + s, step 0.157, 10 leapfrog steps, unit mass) must be
    N(0,1) by the reference's C3 criteria."""
    from math import erf
    d = pcv.Dataset(np.array([0.0, 1.0]), np.zeros((2, 1)))
    f = pcv.make_loo_scheme(d)
    m = pcv.LogisticModel("N01", d, f)
    kp = pcv.KernelParams(0.157, 10, np.array([1.0, 1.0]))
    ks_pass, worst_z, worst_var = 0, 0.0, 0.0
    with pcv.Context(0) as c:
        slot = c.add_model(m, kp, np.zeros((4, 2)), model_id=0)
        for seed in range(10):
            chains = []
            for ch in range(4):
                traj, div = c.hmc_chain(slot, 0, ch, 3000 + seed, np.zeros(2), 10000)
                chains.append(traj[:, 1])
            pooled = np.concatenate(chains)
            mean, var = pooled.mean(), pooled.var(ddof=1)
            mcse = np.sqrt(batch_means_variance(chains, 100) / pooled.size)
            worst_z = max(worst_z, abs(mean) / mcse)
            worst_var = max(worst_var, abs(var - 1.0))
            xs = np.sort(pooled)
            cdf = 0.5 * (1.0 + np.array([erf(v / np.sqrt(2.0)) for v in xs]))
            i = np.arange(xs.size)
            dstat = max(np.max(np.abs(cdf - (i + 1) / xs.size)), np.max(np.abs(cdf - i / xs.size)))
            ks_pass += dstat < 1.6276 / np.sqrt(xs.size)
    print(f"C3: KS passes {ks_pass}/10, worst |mean|/MCSE {worst_z:.2f}, worst |var-1| {worst_var:.3f}")
    assert ks_pass >= 9 and worst_z <= 3.0 and worst_var <= 0.10


# ------------------------------------------------------------------------------ C5
def test_example1_selection_c5():
    prob_ok, ordering_ok, probs = 0, True, []
    for seed in range(10):
        d = pcv.simulate_grouped_regression(50, 5, 4, 1.0, seed=500 + seed)
        f = pcv.make_logo_scheme(d)
        ma = pcv.GroupedRegressionModel("M_A", d, f, [1, 1, 1, 1])
        mb = pcv.GroupedRegressionModel("M_B", d, f, [1, 1, 1, 0])
        with pcv.Context(0) as c:
            acfg = pcv.AdaptConfig(chains=4, warmup=800, draws=1000, n_leapfrog=16)
            fits = [c.adapt_full_data(mm, acfg, seed=9000 + seed, model_id=i) for i, mm in enumerate((ma, mb))]
            for i, (mm, fit) in enumerate(zip((ma, mb), fits)):
                c.add_model(mm, fit.kparams, fit.draws, model_id=i)
            rep = c.run(abi.run_config(chains=4, iters=1000, warmup=100, batch_size=50, blocks=5, bench_draws=50,
                                       checkpoint_every=500, seed=9000 + seed))
        probs.append(rep["prob_a_better"])
        prob_ok += rep["prob_a_better"] > 0.9
        for snap in rep["snapshots"]:
            if snap[0] >= 500 and not snap[2] < snap[3]:
                ordering_ok = False
    print(f"C5: prob > 0.9 on {prob_ok}/10 seeds (min {min(probs):.3f})")
    assert prob_ok >= 8 and ordering_ok


# ------------------------------------------------------------------------------ failed folds
@pytest.mark.parametrize("name,broken,policy", [("cfg1_linreg_loo", 0, None), ("cfg1_linreg_loo", 0, "rows"),
                                                ("ex1_grouped_logo", 1, None), ("radon_logo", 0, "rows"),
                                                ("logistic_loo", 0, None)])
def test_failed_fold_excluded_but_reported(name, broken, policy):
    """BrokenFoldModel on fold 3 of one model (test_engine.cpp:240-255): every chain of that fold
    diverges on every transition, the fold is failed and excluded for both models (engine.cpp:
    385-397), its divergences are reported, delta-hat sums the remaining folds, and the shuffle
    benchmark runs over the non-failed folds only - the same failed flags, divergence counts and
    (at this short horizon, on the same streams) benchmark replicates as the oracle."""
    case = Case(name)
    fold = 3
    c = pcv.Context(0)
    if policy == "rows":
        c.set_kernel_policy(c.KERNEL_ROWS)
    slots = [c.add_model(m, kp, bank, model_id=i)
             for i, (m, kp, bank) in enumerate(zip(case.models, case.kparams, case.banks))]
    c.debug_break_fold(slots[broken], fold)
    case.omodels[broken].break_fold(fold)
    cfg = abi.run_config(chains=4, iters=12, warmup=3, batch_size=3, blocks=4, bench_draws=20, seed=5)
    rep = c.run(cfg)
    c.close()
    orep = O.run_pcv_oracle(case.omodels, list(range(len(case.omodels))),
                            [abi.KernelArrays(k.step_size, k.n_leapfrog, k.inv_mass_diag) for k in case.kparams],
                            case.banks, cfg)
    K, L, nm = case.K, 4, len(case.models)
    failed = rep["failed"].reshape(nm, K)
    assert np.array_equal(failed, orep["failed"].reshape(nm, K))
    assert all(np.flatnonzero(failed[m]).tolist() == [fold] for m in range(nm))
    div = rep["divergences"].reshape(nm, K, L)
    assert np.all(div[broken, fold] == cfg.iters)
    np.testing.assert_array_equal(rep["divergences"], orep["divergences"])
    keep = np.ones(K, bool)
    keep[fold] = False
    assert rep["delta_hat"] == pytest.approx(np.sum(rep["delta_k"][keep]), rel=1e-13, abs=1e-12)
    assert rep["benchmark_count"] == orep["benchmark_count"]
    np.testing.assert_allclose(rep["benchmark"], orep["benchmark"], rtol=1e-8)
    np.testing.assert_allclose(rep["delta_hat"], orep["delta_hat"], rtol=1e-8)

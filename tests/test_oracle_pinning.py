"""Pins the CPU oracle (oracle/pcv_oracle.c) - the checker every GPU parity test uses.

(a) Golden vectors and closed forms from the reference's own test suite (always run; they need
    neither the reference sources nor a GPU).
(b) Bit-for-bit agreement with the reference library compiled in place (`ref` marker; runs where
    oracle/_ref/libpcvref.so exists, i.e. in the build container).
(c) The committed reference fixtures (tests/golden/*.npz, generated from the reference by
    make_golden.py): the oracle's run_pcv reproduces the reference report bit for bit.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2310_07002_b200 import abi
import _oracle as O
from parity_util import ALL_FIXTURES, Case, sample_thetas

LIB = O.oracle()


def seq(lib_fn, seed, stream, ops, args=None, skip=None):
    ops_b = ops.encode()
    arg = np.zeros(len(ops_b), dtype=np.uint64) if args is None else np.asarray(args, dtype=np.uint64)
    out = np.zeros(len(ops_b))
    rc = lib_fn(seed, stream, int(skip is not None), skip or 0, ops_b, abi.ptr(arg, C.c_uint64), len(ops_b),
                abi.ptr(out, C.c_double))
    assert rc == 0
    return out


# ---------------------------------------------------------------- (a) golden vectors
PHILOX_KATS = [  # test_rng.cpp:15-23 (Salmon et al.)
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("kat", PHILOX_KATS)
def test_philox_known_answers(kat):
    ctr, key, expect = kat
    seed = key[0] | (key[1] << 32)
    stream = ctr[2] | (ctr[3] << 32)
    out = seq(LIB.pcvo_rng_sequence, seed, stream, "4444", skip=ctr[0] | (ctr[1] << 32))
    assert [int(v) for v in out] == list(expect)


def test_streams_deterministic_and_independent():  # test_rng.cpp:36-47
    k1 = LIB.pcvo_stream_key(abi.STREAM_CHAIN_SAMPLING, 0, 3, 1)
    k2 = LIB.pcvo_stream_key(abi.STREAM_CHAIN_SAMPLING, 0, 3, 2)
    a = seq(LIB.pcvo_rng_sequence, 42, k1, "4" * 200)
    b = seq(LIB.pcvo_rng_sequence, 42, k1, "4" * 200)
    c = seq(LIB.pcvo_rng_sequence, 42, k2, "4" * 200)
    assert np.array_equal(a, b)
    assert len(set(c.tolist())) == 200 and not np.array_equal(a, c)


def test_uniform_normal_moments():  # test_rng.cpp:49-67
    n = 200000
    u = seq(LIB.pcvo_rng_sequence, 7, 1, "u" * n)
    z = seq(LIB.pcvo_rng_sequence, 7, 2, "n" * n)
    assert u.min() > 0 and u.max() < 1
    assert abs(u.mean() - 0.5) < 0.005 and abs(u.var() - 1 / 12) < 0.05 / 12
    assert abs(z.mean()) < 0.01 and abs(z.var() - 1) < 0.02


def test_below_uniform():  # test_rng.cpp:69-74
    b = seq(LIB.pcvo_rng_sequence, 9, 2, "b" * 70000, args=np.full(70000, 7))
    counts = np.bincount(b.astype(int), minlength=7)
    assert np.all(np.abs(counts - 10000) < 500)


def test_kfold_sizes_and_determinism():  # test_folds_dataset.cpp:59-79
    def kf(n, K, seed):
        out = np.zeros(n, dtype=np.int32)
        rc = LIB.pcvo_make_kfold(n, K, seed, abi.ptr(out, C.c_int32))
        return rc, out
    rc, f10 = kf(10, 5, 3)
    assert rc == 0 and all(np.sum(f10 == k) == 2 for k in range(5))
    rc, f11 = kf(11, 5, 3)
    assert sorted(np.bincount(f11)) == [2, 2, 2, 2, 3]
    assert np.array_equal(kf(11, 5, 3)[1], f11) and not np.array_equal(kf(11, 5, 4)[1], f11)
    assert kf(10, 1, 3)[0] != 0 and kf(10, 11, 3)[0] != 0


def test_time_blocks_contiguous():  # test_folds_dataset.cpp:81-93
    t = np.array([16 - i for i in range(17)], dtype=np.int64)
    d = abi.DatasetArrays(np.arange(17.0), None, None, t)
    out = np.zeros(17, dtype=np.int32)
    assert LIB.pcvo_make_time_blocks(C.byref(d.struct), 4, abi.ptr(out, C.c_int32)) == 0
    by_time = np.empty(17, dtype=np.int32)
    by_time[t] = out
    assert np.all(np.diff(by_time) >= 0)


def test_hv_block_geometry():
    n, K, h = 598, 20, 6
    d = abi.DatasetArrays(np.zeros(n), None, None, np.arange(n, dtype=np.int64))
    iv = np.zeros(4 * K, dtype=np.int64)
    assert LIB.pcvo_make_hv_block(C.byref(d.struct), K, h, abi.ptr(iv, C.c_int64)) == 0
    iv = iv.reshape(K, 4)
    assert iv[0, 0] == 0 and iv[-1, 1] == n and np.all(iv[1:, 0] == iv[:-1, 1])  # test blocks partition
    assert np.all(iv[:, 2] == np.maximum(0, iv[:, 0] - h)) and np.all(iv[:, 3] == np.minimum(n, iv[:, 1] + h))
    iv2 = np.zeros(4 * n, dtype=np.int64)
    assert LIB.pcvo_make_hv_racine(C.byref(d.struct), 5, 3, abi.ptr(iv2, C.c_int64)) == 0
    iv2 = iv2.reshape(n, 4)
    t = 100
    assert tuple(iv2[t]) == (95, 106, 92, 109)


def test_rhat_closed_forms():  # test_diagnostics.cpp:21-41, acceptance C2
    w, b, r = C.c_double(), C.c_double(), C.c_double()
    sx = np.array([3.0, 7.0])
    sxx = np.array([5.0, 25.0])
    assert LIB.pcvo_rhat_from_sums(abi.ptr(sx, C.c_double), abi.ptr(sxx, C.c_double), 2, 2,
                                   C.byref(w), C.byref(b), C.byref(r)) == 1
    assert abs(w.value - 0.5) < 1e-12 and abs(b.value - 4.0) < 1e-12 and abs(r.value - np.sqrt(4.5)) < 1e-12
    ch = np.array([0.1, -0.4, 0.9, 1.3, -0.2])
    sx = np.full(3, ch.sum())
    sxx = np.full(3, (ch ** 2).sum())
    assert LIB.pcvo_rhat_from_sums(abi.ptr(sx, C.c_double), abi.ptr(sxx, C.c_double), 3, 5,
                                   C.byref(w), C.byref(b), C.byref(r)) == 1
    assert abs(b.value) < 1e-12 and abs(r.value - np.sqrt(4 / 5)) < 1e-12
    sx, sxx = np.array([4.0, 4.0]), np.array([8.0, 8.0])  # constant chains -> undefined
    assert LIB.pcvo_rhat_from_sums(abi.ptr(sx, C.c_double), abi.ptr(sxx, C.c_double), 2, 2,
                                   C.byref(w), C.byref(b), C.byref(r)) == 0


def test_selection_probability():  # test_scoring.cpp:201-238
    s2 = C.c_double()
    d = np.array([0.5, -0.5, 0.25, -0.25])
    assert abs(LIB.pcvo_selection_probability(0.0, abi.ptr(d, C.c_double), 4, C.byref(s2)) - 0.5) < 1e-12
    k, sigma2 = 4.0, 4.0 / 3.0
    target = 2.0 * np.sqrt(k * sigma2)
    shifted = np.array([1.0, -1.0, 1.0, -1.0]) + target / k
    p = LIB.pcvo_selection_probability(target, abi.ptr(shifted, C.c_double), 4, C.byref(s2))
    assert abs(p - 0.9772498680518208) < 1e-5
    eq = np.array([1.0, 1.0])
    assert LIB.pcvo_selection_probability(2.0, abi.ptr(eq, C.c_double), 2, C.byref(s2)) == 1.0


def test_benchmark_nearest_rank():  # test_diagnostics.cpp:99-110
    v = 1.0 + 0.001 * np.arange(1, 101)
    q = LIB.pcvo_benchmark_quantile(abi.ptr(v, C.c_double), 100, 0.99)
    assert abs(q - 1.099) < 1e-12


def score_streams(streams, center, b, D):
    s = np.ascontiguousarray(np.atleast_2d(streams), dtype=np.float64)
    out = np.zeros(8)
    assert LIB.pcvo_score_streams(s.shape[0], s.shape[1], abi.ptr(s, C.c_double), center, b, D,
                                  abi.ptr(out, C.c_double)) == 0
    return out


def two_pass(chains, batch):
    """Stored-draw oracle (test_support.hpp:29-88) in extended precision."""
    ch = np.asarray(chains, dtype=np.longdouble)
    f = np.exp(ch)
    ln = f.size
    fhat = f.mean()
    s2 = ((f - fhat) ** 2).sum() / (ln - 1)
    a = ch.shape[1] // batch
    bm = f[:, :a * batch].reshape(ch.shape[0], a, batch).mean(axis=2)
    sigma2 = batch * ((bm - fhat) ** 2).sum() / (ch.shape[0] * a - 1)
    return float(np.log(fhat)), float(s2 / fhat ** 2), float(sigma2 / fhat ** 2)


def test_logs_closed_cases():  # test_scoring.cpp:12-42
    logc = np.log(0.37)
    out = score_streams(np.full((2, 100), logc), logc, 10, 5)
    assert abs(out[0] - logc) < 1e-12 * abs(logc) and abs(out[2]) < 1e-12
    out = score_streams([[np.log(0.5), np.log(1.5)]], 0.0, 1, 1)
    assert abs(out[0]) < 1e-14
    out = score_streams(np.full((1, 20), -np.inf), 0.0, 5, 2)
    assert out[0] == -np.inf and out[7] == 1 and np.isinf(out[2])


def test_online_equals_two_pass():  # test_accum.cpp:180-202, acceptance C1
    rng = np.random.default_rng(2)
    for trial in range(10):
        ch = -2.0 + 0.8 * rng.standard_normal((4, 900))
        out = score_streams(ch, -2.0, 50, 5)
        ref_score, ref_naive, ref_mc = two_pass(ch, 50)
        assert abs(out[0] - ref_score) <= 1e-10 * abs(ref_score)
        assert abs(out[3] - ref_naive) <= 1e-8 * ref_naive
        assert abs(out[2] - ref_mc) <= 1e-8 * ref_mc


def test_fd_gradients_all_families():  # test_models.cpp:17-34 (rel 1e-4)
    for name in ALL_FIXTURES:
        case = Case(name)
        for m, om in enumerate(case.omodels):
            for fold in [0, case.K // 2, case.K]:
                th = sample_thetas(case, m, 2, seed=fold)
                for t in th:
                    g = om.grad(t, fold)
                    fd = np.zeros_like(g)
                    for i in range(len(t)):
                        h = 1e-5 * max(1.0, abs(t[i]))
                        tp, tm = t.copy(), t.copy()
                        tp[i] += h
                        tm[i] -= h
                        fd[i] = (om.log_joint(tp, fold) - om.log_joint(tm, fold)) / (2 * h)
                    scale = np.maximum(1.0, np.abs(g))
                    assert np.max(np.abs(fd - g) / scale) < 1e-4, (name, m, fold)


# ---------------------------------------------------------------- (c) reference fixtures
@pytest.mark.parametrize("name", ALL_FIXTURES)
def test_oracle_reproduces_reference_report(name):
    """Oracle run_pcv on the fixture inputs == the reference run_pcv report stored by make_golden.py
    (same Philox streams, same arithmetic order): bit-identical headline statistics."""
    case = Case(name)
    z = case.z
    rc = z["run_cfg"]
    cfg = abi.run_config(chains=int(rc[0]), iters=int(rc[1]), warmup=int(rc[2]), batch_size=int(rc[3]),
                         blocks=int(rc[4]), bench_draws=int(rc[5]), checkpoint_every=int(rc[6]), seed=1)
    rep = O.run_pcv_oracle(case.omodels, list(range(len(case.omodels))),
                           [abi.KernelArrays(k.step_size, k.n_leapfrog, k.inv_mass_diag) for k in case.kparams],
                           case.banks, cfg, threads=4)
    for k in ("delta_hat", "mcse", "sigma2_delta", "epistemic_se", "ess_overall", "rhat_max"):
        assert rep[k] == float(z[f"ref_{k}"]) or (np.isnan(rep[k]) and np.isnan(z[f"ref_{k}"])), k
    np.testing.assert_array_equal(rep["estimate"], z["ref_estimate"])
    np.testing.assert_array_equal(rep["rhat"], z["ref_rhat"])
    np.testing.assert_array_equal(rep["divergences"], z["ref_divergences"])
    np.testing.assert_array_equal(rep["benchmark"], z["ref_benchmark"])
    np.testing.assert_array_equal(rep["snapshots"], z["ref_snapshots"])


# ---------------------------------------------------------------- (b) reference library itself
@pytest.mark.ref
def test_rng_matches_reference():
    R = O.ref()
    ops = "nnnunn4bnunnnnnuu" * 40
    args = np.where(np.array(list(ops)) == "b", 13, 0).astype(np.uint64)
    for seed, stream in [(1, 2), (5, 9), (2 ** 40 + 3, 7)]:
        a = seq(LIB.pcvo_rng_sequence, seed, stream, ops, args)
        b = seq(R.pcvref_rng_sequence, seed, stream, ops, args)
        assert np.array_equal(a, b)
    for args_ in [(1, 0, 3, 1), (2, 1, 99, 7), (6, 250, 0, 0)]:
        assert LIB.pcvo_stream_key(*args_) == R.pcvref_stream_key(*args_)


@pytest.mark.ref
def test_folds_match_reference():
    R = O.ref()
    for n, K, seed in [(11, 5, 3), (1000, 10, 1), (4998, 100, 7)]:
        a, b = np.zeros(n, np.int32), np.zeros(n, np.int32)
        LIB.pcvo_make_kfold(n, K, seed, abi.ptr(a, C.c_int32))
        R.pcvref_make_kfold(n, K, seed, abi.ptr(b, C.c_int32))
        assert np.array_equal(a, b)
    t = np.random.default_rng(0).permutation(500).astype(np.int64)
    d = abi.DatasetArrays(np.zeros(500), None, None, t)
    a, b = np.zeros(500, np.int32), np.zeros(500, np.int32)
    LIB.pcvo_make_time_blocks(C.byref(d.struct), 17, abi.ptr(a, C.c_int32))
    R.pcvref_make_time_blocks(C.byref(d.struct), 17, abi.ptr(b, C.c_int32))
    assert np.array_equal(a, b)


@pytest.mark.ref
@pytest.mark.parametrize("name", ALL_FIXTURES)
def test_models_match_reference_bitwise(name):
    case = Case(name)
    for m, om in enumerate(case.omodels):
        rm = O.RModel(case.data, case.fa, abi.SpecArrays(**case.kws[m]))
        for fold in sorted({0, 1, case.K // 2, case.K - 1, case.K}):
            for t in sample_thetas(case, m, 3, seed=fold):
                assert om.log_joint(t, fold) == rm.log_joint(t, fold)
                assert np.array_equal(om.grad(t, fold), rm.grad(t, fold))
                assert om.log_pred(t, fold) == rm.log_pred(t, fold)


@pytest.mark.ref
@pytest.mark.parametrize("name", ["cfg1_linreg_loo", "radon_logo", "seasonal_hvblock", "logistic_loo"])
def test_partition_identity(name):  # test_models.cpp:36-47 on the reference, oracle log_joint
    case = Case(name)
    rm = O.RModel(case.data, case.fa, abi.SpecArrays(**case.kws[0]))
    t = sample_thetas(case, 0, 1, seed=4)[0]
    full = case.omodels[0].log_joint(t, case.K)
    if case.folds.intervals is not None:
        pytest.skip("hv-block folds do not partition the likelihood (gap rows)")
    for k in range(0, case.K, max(1, case.K // 17)):
        s = case.omodels[0].log_joint(t, k) + rm.log_lik_test(t, k)
        assert abs(s - full) <= 1e-10 * abs(full)


@pytest.mark.ref
@pytest.mark.parametrize("name", ALL_FIXTURES)
def test_hmc_trajectory_matches_reference_bitwise(name):
    case = Case(name)
    om, kp = case.omodels[0], case.kparams[0]
    rm = O.RModel(case.data, case.fa, abi.SpecArrays(**case.kws[0]))
    stream = LIB.pcvo_stream_key(abi.STREAM_CHAIN_SAMPLING, 0, 1, 2)
    th0 = case.banks[0][5]
    a, da = om.hmc_chain(1, kp.step_size, kp.n_leapfrog, kp.inv_mass_diag, 3, stream, th0, 40)
    b, db = rm.hmc_chain(1, kp.step_size, kp.n_leapfrog, kp.inv_mass_diag, 3, stream, th0, 40)
    assert np.array_equal(a, b) and np.array_equal(da, db)


# ---------------------------------------------------------------- HS / DSS (engine.cpp:322-373)
SCORE_CASES = [(base, sc) for base in ["cfg1_linreg_loo", "ex1_grouped_logo", "radon_logo",
                                       "seasonal_timeblocks", "seasonal_hvblock", "rat_logo"]
               for sc in ("hs", "dss")]


def score_fixture(base, sc):
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", f"{base}_{sc}.npz"))
    return z


@pytest.mark.parametrize("base,sc", SCORE_CASES)
def test_oracle_reproduces_reference_score_report(base, sc):
    """Oracle run_pcv with score HS / DSS == the reference run_pcv report (make_golden.py
    make_score): same chain streams (DSS draws consume them), same Welford arithmetic, same
    hs_fold_score / dss_fold_score."""
    case = Case(base)
    z = score_fixture(base, sc)
    rc = case.z["run_cfg"]
    cfg = abi.run_config(chains=int(rc[0]), iters=int(rc[1]), warmup=int(rc[2]), batch_size=int(rc[3]),
                         blocks=int(rc[4]), bench_draws=int(rc[5]), checkpoint_every=int(rc[6]), seed=1,
                         score=int(z["score"]))
    rep = O.run_pcv_oracle(case.omodels, list(range(len(case.omodels))),
                           [abi.KernelArrays(k.step_size, k.n_leapfrog, k.inv_mass_diag) for k in case.kparams],
                           case.banks, cfg, threads=4)
    for k in ("delta_hat", "sigma2_delta", "epistemic_se", "ess_overall", "rhat_max"):
        assert rep[k] == float(z[f"ref_{k}"]) or (np.isnan(rep[k]) and np.isnan(z[f"ref_{k}"])), k
    assert np.isnan(rep["mcse"]) and np.isnan(z["ref_mcse"])  # MCSE is LogS-only
    np.testing.assert_array_equal(rep["estimate"], z["ref_estimate"])
    np.testing.assert_array_equal(rep["fault"], z["ref_fault"])
    np.testing.assert_array_equal(rep["dss_ridged"], z["ref_dss_ridged"])
    np.testing.assert_array_equal(rep["divergences"], z["ref_divergences"])
    np.testing.assert_array_equal(rep["snapshots"], z["ref_snapshots"])


def test_hs_closed_forms():  # test_scoring.cpp:44-62 via the oracle's pred_derivs on a 1-row fold
    case = Case("cfg1_linreg_loo")
    om = case.omodels[0]
    th = case.banks[0][3].copy()
    d1, d2 = om.pred_derivs(th, 7)
    vy = np.exp(th[-1]) ** 2
    mean = th[0] + case.data.x[7] @ th[1:6]
    assert d2[0] == -1.0 / vy
    assert abs(d1[0] + (case.data.y[7] - mean) / vy) <= 1e-13 * abs(d1[0])
    # HS of a point mass at the predictive derivatives: 2(d2 + d1^2) - d1^2 (scoring.cpp:64-73)


@pytest.mark.ref
@pytest.mark.parametrize("name", ["cfg1_linreg_loo", "ex1_grouped_logo", "radon_logo",
                                  "seasonal_timeblocks", "seasonal_hvblock", "rat_logo"])
def test_pred_hooks_match_reference_bitwise(name):
    """Model::pred_derivs / pred_sample of the oracle == the reference (same stream)."""
    case = Case(name)
    for m, om in enumerate(case.omodels):
        rm = O.RModel(case.data, case.fa, abi.SpecArrays(**case.kws[m]))
        for fold in sorted({0, 1, case.K // 2, case.K - 1}):
            for t in sample_thetas(case, m, 2, seed=fold):
                a1, a2 = om.pred_derivs(t, fold)
                b1, b2 = rm.pred_derivs(t, fold)
                assert np.array_equal(a1, b1) and np.array_equal(a2, b2)
                assert np.array_equal(om.pred_sample(t, fold, 3, 11, 3), rm.pred_sample(t, fold, 3, 11, 3))


@pytest.mark.ref
@pytest.mark.parametrize("name", ["cfg1_linreg_loo", "ex1_grouped_logo", "radon_logo", "seasonal_timeblocks",
                                  "seasonal_hvblock", "logistic_loo", "rat_logo"])
def test_initial_draw_matches_reference_bitwise(name):
    """pcvg_initial_draw (host, the full-data chains' starts) == Model::initial_draw of the
    reference (grouped_regression.cpp:177-188, radon.cpp:157-165, seasonal_ar.cpp:122-131)."""
    from paper_2310_07002_b200 import pcv
    case = Case(name)
    for m, model in enumerate(case.models):
        rm = O.RModel(case.data, case.fa, abi.SpecArrays(**case.kws[m]))
        for c in range(4):
            st = pcv.stream_key(abi.STREAM_FULL_DATA, m, c)
            assert np.array_equal(pcv.initial_draw(model, 7, st), rm.initial_draw(7, st))


@pytest.mark.ref
def test_adapt_trace_oracle_matches_reference():
    """The traced restatement of adapt_full_data (ref_shim pcvref_adapt_trace, used to pin the
    device adaptation step by step) reproduces the reference's own inverse mass."""
    z = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "adapt_short.npz"))
    for name in ("cfg1_linreg_loo", "radon_logo"):
        case = Case(name)
        rm = O.RModel(case.data, case.fa, abi.SpecArrays(**case.kws[0]))
        tr = rm.adapt_trace(chains=4, warmup=30, seed=3, model_id=0)
        assert np.array_equal(tr["inv_mass"], z[f"{name}:0:inv_mass"])
        assert np.array_equal(tr["step_trace"], z[f"{name}:0:step_trace"])


# ---------------------------------------------------------------- bench.py CPU arms
def test_refarm_builds_cfg2_without_the_product_library():
    """bench.py's reference arm (oracle/refarm.py) simulates the cfg2 dataset inside the CPU library
    (the reference plugin's simulator, or the oracle port's); both must equal the product simulator
    bit for bit, and the arm must not load libpcvg.so."""
    import os
    import subprocess
    import sys
    from paper_2310_07002_b200 import pcv
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import refarm
    d = pcv.simulate_logistic(2000, 50, seed=1)
    for prefer_ref in ([True, False] if O.have_ref() else [False]):
        w = refarm.Workload(prefer_ref)
        y, x = np.zeros(2000), np.zeros(2000 * 50)
        sim = w.lib.pcvref_simulate_logistic if w.kind == "reference" else w.lib.pcvo_simulate_logistic
        sim.argtypes = [C.c_int64, C.c_int32, C.c_uint64, refarm.PF64, refarm.PF64]
        assert sim(2000, 50, 1, refarm._ptr(y, C.c_double), refarm._ptr(x, C.c_double)) == 0
        assert np.array_equal(y, d.y) and np.array_equal(x.reshape(d.x.shape), d.x), w.kind
        w.close()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, 'oracle'); import refarm; w = refarm.Workload(); "
            "maps = open('/proc/self/maps').read(); print('libpcvg' in maps, 'paper_2310_07002_b200' in sys.modules)")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.split() == ["False", "False"]

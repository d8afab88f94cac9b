"""CPU-side tests of the product library libpcvg.so (no GPU needed): the C ABI exports, the
bit-exact host restatements (Philox, fold schemes, simulators) and the Step-4 host merge, which is
checked against the oracle's compute_stats on a full oracle run."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2310_07002_b200 import abi, pcv
import _oracle as O
from parity_util import Case

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "pcvg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pcvg_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(abi.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert pcv.load().pcvg_abi_version() == abi.ABI_VERSION


def test_status_names():
    lib = pcv.load()
    assert lib.pcvg_status_name(abi.INVALID_INPUT) == b"invalid_input"
    assert lib.pcvg_status_name(abi.UNSUPPORTED_SCORE) == b"unsupported_score"


def test_no_cpu_fallback():
    """Device entry points fail loudly without a GPU (there is no CPU path in the product)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pcv.CudaError):
        pcv.Context(0)


def test_philox_and_streams_match_oracle():
    L = O.oracle()
    ops = "nnunn4bnuu" * 50
    args = np.where(np.array(list(ops)) == "b", 11, 0).astype(np.uint64)
    for seed, stream in [(1, 2), (2 ** 33 + 5, 77)]:
        a = pcv.rng_sequence(seed, stream, ops, args)
        b = np.zeros(len(ops))
        L.pcvo_rng_sequence(seed, stream, 0, 0, ops.encode(), abi.ptr(args, C.c_uint64), len(ops),
                            abi.ptr(b, C.c_double))
        assert np.array_equal(a, b)
    # KAT through the product (test_rng.cpp:15-23)
    out = pcv.rng_sequence(0xFFFFFFFFFFFFFFFF, 0xFFFFFFFFFFFFFFFF, "4444", skip_block=0xFFFFFFFFFFFFFFFF)
    assert [int(v) for v in out] == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert pcv.stream_key(1, 2, 3, 4) == L.pcvo_stream_key(1, 2, 3, 4)


def test_fold_schemes_match_oracle():
    L = O.oracle()
    for n, K, seed in [(11, 5, 3), (10000, 10, 1)]:
        f = pcv.make_kfold_scheme(n, K, seed)
        o = np.zeros(n, np.int32)
        L.pcvo_make_kfold(n, K, seed, abi.ptr(o, C.c_int32))
        assert np.array_equal(f.test_index, o)
    d = pcv.simulate_seasonal_ar(600, 2, 11, 0.6, seed=7)
    f = pcv.make_time_block_scheme(d, 20)
    o = np.zeros(d.n_obs, np.int32)
    L.pcvo_make_time_blocks(C.byref(d.struct), 20, abi.ptr(o, C.c_int32))
    assert np.array_equal(f.test_index, o)
    for maker, args in ((pcv.make_hv_block_scheme, (20, 6)), (pcv.make_hv_racine_scheme, (5, 3))):
        f = maker(d, *args)
        o = np.zeros_like(f.intervals)
        fn = L.pcvo_make_hv_block if maker is pcv.make_hv_block_scheme else L.pcvo_make_hv_racine
        fn(C.byref(d.struct), *args, abi.ptr(o, C.c_int64))
        assert np.array_equal(f.intervals, o)
    loo = pcv.make_loo_scheme(d)
    assert loo.K == d.n_obs and np.array_equal(loo.test_index, np.arange(d.n_obs))
    g = pcv.simulate_grouped_regression(50, 5, 4, 1.0, seed=1)
    logo = pcv.make_logo_scheme(g)
    assert logo.K == 50 and np.array_equal(logo.test_index, g.group_id)


def test_fold_scheme_errors():  # folds.cpp preconditions -> invalid_input
    with pytest.raises(pcv.InvalidInput):
        pcv.make_kfold_scheme(10, 1, 3)
    with pytest.raises(pcv.InvalidInput):
        pcv.make_kfold_scheme(10, 11, 3)
    with pytest.raises(pcv.InvalidInput):
        pcv.make_loo_scheme(pcv.Dataset(np.zeros(1)))
    with pytest.raises(pcv.InvalidInput):
        pcv.make_logo_scheme(pcv.Dataset(np.zeros(3), None, np.zeros(3, np.int32)))
    with pytest.raises(pcv.InvalidInput):
        pcv.make_time_block_scheme(pcv.Dataset(np.zeros(5)), 2)


@pytest.mark.ref
def test_simulators_match_reference_bitwise():
    R = O.ref()
    d = pcv.simulate_grouped_regression(50, 5, 4, 1.0, seed=1)
    y, x, g = np.zeros(250), np.zeros(1000), np.zeros(250, np.int32)
    R.pcvref_simulate_grouped(50, 5, 4, 1.0, 1, abi.ptr(y, C.c_double), abi.ptr(x, C.c_double), abi.ptr(g, C.c_int32))
    assert np.array_equal(d.y, y) and np.array_equal(d.x.ravel(), x) and np.array_equal(d.group_id, g)
    d = pcv.simulate_radon_style(12000, 400, 5)
    y, x, g = np.zeros(12000), np.zeros(12000), np.zeros(12000, np.int32)
    R.pcvref_simulate_radon(12000, 400, 5, abi.ptr(y, C.c_double), abi.ptr(x, C.c_double), abi.ptr(g, C.c_int32))
    assert np.array_equal(d.y, y) and np.array_equal(d.x.ravel(), x) and np.array_equal(d.group_id, g)
    d = pcv.simulate_seasonal_ar(5000, 2, 11, 0.6, seed=7)
    n = 4998
    y, x, t = np.zeros(n), np.zeros(n * 13), np.zeros(n, np.int64)
    R.pcvref_simulate_seasonal(5000, 2, 11, 0.6, 1.0, 1.0, 7, abi.ptr(y, C.c_double), abi.ptr(x, C.c_double),
                               abi.ptr(t, C.c_int64))
    assert np.array_equal(d.y, y) and np.array_equal(d.x.ravel(), x) and np.array_equal(d.time_index, t)


def _oracle_run(case, cfg):
    """Oracle run_pcv + its per-task accumulators (for the block sums)."""
    L = O.oracle()
    nm = len(case.omodels)
    K, Lc, D = case.K, cfg.chains, cfg.blocks
    ntask = nm * K * Lc
    stride = 10 + 2 * D
    accum = np.zeros(ntask * stride)
    dimmax = max(m.dim for m in case.omodels)
    pos = np.zeros(ntask * dimmax)
    warm = np.zeros(ntask)
    divs = np.zeros(ntask, np.int64)

    class TaskOut(C.Structure):
        _fields_ = [("position", abi.P_f64), ("warm_logpred", abi.P_f64), ("divergences", abi.P_i64),
                    ("accum", abi.P_f64)]
    tout = TaskOut(abi.ptr(pos, C.c_double), abi.ptr(warm, C.c_double), abi.ptr(divs, C.c_int64),
                   abi.ptr(accum, C.c_double))
    rep, arrs = abi.new_report(nm, K, Lc, abi.checkpoint_count(cfg.iters, cfg.checkpoint_every), cfg.bench_draws)
    arr_h = (C.c_void_p * nm)(*[m.h for m in case.omodels])
    kerns = [abi.KernelArrays(k.step_size, k.n_leapfrog, k.inv_mass_diag) for k in case.kparams]
    ks = (abi.Kernel * nm)(*[k.struct for k in kerns])
    banks = [np.ascontiguousarray(b) for b in case.banks]
    bptr = (abi.P_f64 * nm)(*[abi.ptr(b, C.c_double) for b in banks])
    rows = np.array([b.shape[0] for b in banks], np.int64)
    ids = np.arange(nm, dtype=np.int32)
    rc = L.pcvo_run_pcv(nm, arr_h, abi.ptr(ids, C.c_int32), ks, bptr, abi.ptr(rows, C.c_int64), C.byref(cfg), 4,
                        C.byref(rep), C.cast(C.pointer(tout), C.c_void_p), dimmax)
    assert rc == 0
    acc = accum.reshape(ntask, stride)
    return abi.report_dict(rep, arrs, nm), acc[:, 10:10 + D].copy(), acc[:, 10 + D:].copy()


@pytest.mark.parametrize("name", ["ex1_grouped_logo", "radon_logo", "logistic_kfold"])
def test_host_merge_equals_oracle_compute_stats(name):
    """pcvg_merge (the product's Step 4, engine.cpp:117-253 + benchmark) on the oracle's per-fold
    table and block sums reproduces the oracle's report bit for bit."""
    case = Case(name)
    rc = case.z["run_cfg"]
    cfg = abi.run_config(chains=int(rc[0]), iters=int(rc[1]), warmup=int(rc[2]), batch_size=int(rc[3]),
                         blocks=int(rc[4]), bench_draws=int(rc[5]), seed=1)
    orep, y_x, y_x2 = _oracle_run(case, cfg)
    nm = len(case.omodels)
    cols = {k: orep[k] for k, _ in abi.FOLD_COLUMNS}
    # failed folds as the engine computes them (engine.cpp:385-397)
    from paper_2310_07002_b200 import dist
    cols["failed"] = dist.failed_from_divergences(orep["divergences"], nm, case.K, cfg.chains, cfg.iters)
    rep = pcv.merge(nm, case.K, cfg, cfg.iters, True, cols, y_x.ravel(), y_x2.ravel())
    for k in ("delta_hat", "mcse", "sigma2_delta", "epistemic_se", "ess_overall", "rhat_max", "verdict_pass",
              "verdict_quantile_value"):
        a, b = rep[k], orep[k]
        assert a == b or (np.isnan(a) and np.isnan(b)), (k, a, b)
    if nm == 2:
        assert rep["prob_a_better"] == orep["prob_a_better"]
    assert rep["score_total"] == orep["score_total"]
    np.testing.assert_array_equal(rep["benchmark"], orep["benchmark"])
    np.testing.assert_array_equal(rep["delta_k"], orep["delta_k"])
    np.testing.assert_array_equal(rep["failed"], orep["failed"])


def test_merge_selection_probability_closed_form():  # test_scoring.cpp:201-212 through pcvg_merge
    K = 4
    cfg = abi.run_config(chains=2, iters=10, batch_size=5, bench_draws=1)
    target = 2.0 * np.sqrt(4.0 * 4.0 / 3.0)
    est_a = np.array([1.0, -1.0, 1.0, -1.0]) + target / K
    cols = {k: np.zeros(2 * K, dtype=dt) for k, dt in abi.FOLD_COLUMNS}
    cols["estimate"][:K] = est_a
    cols["rhat"][:] = 1.0
    rep = pcv.merge(2, K, cfg, 10, False, cols)
    assert abs(rep["prob_a_better"] - 0.9772498680518208) < 1e-5
    assert abs(rep["delta_hat"] - target) < 1e-12


def test_merge_rejects_bad_arguments():
    cfg = abi.run_config(chains=2, iters=10, batch_size=5)
    cols = {k: np.zeros(2, dtype=dt) for k, dt in abi.FOLD_COLUMNS}
    with pytest.raises(pcv.InvalidInput):
        pcv.merge(3, 2, cfg, 10, False, {k: np.zeros(6, dtype=dt) for k, dt in abi.FOLD_COLUMNS})
    with pytest.raises(pcv.InvalidInput):
        pcv.merge(1, 1, cfg, 10, False, cols)


@pytest.mark.parametrize("scheme", ["loo", "kfold", "hv"])
def test_fold_gram_is_the_rounded_exact_training_sum(scheme):
    """Fold statistics of the sufficient-statistics kernel (suffstats.cpp): every
    packed Gram entry of every fold is the training-row sum of u u^T (u = (y, x)) formed as
    full - excluded in double-double, i.e. the exact rational sum rounded once (here: within
    one ulp of it, also when cancellation makes the training sum tiny)."""
    from fractions import Fraction
    rng = np.random.default_rng(4)
    n, nc = 40, 3
    x = rng.standard_normal((n, nc)) * np.array([1.0, 1e3, 1e-3])
    y = 1e4 + rng.standard_normal(n)  # large mean: sum y^2 cancels strongly in full - excluded
    if scheme == "loo":
        key = np.arange(n, dtype=np.int32)
        lo, hi = np.arange(n), np.arange(n) + 1
    elif scheme == "kfold":
        key = rng.integers(0, 5, n).astype(np.int32)
        lo, hi = np.arange(5), np.arange(5) + 1
    else:  # hv-block: key = time rank, exclusion windows
        key = rng.permutation(n).astype(np.int32)
        lo = np.array([0, 5, 30, 35]); hi = np.array([12, 17, 40, 40])
    g = pcv.fold_gram(y, x, key, lo, hi)
    u = np.column_stack([y, x])
    K = lo.size
    fu = [[Fraction(float(v)) for v in row] for row in u]
    for k in range(K + 1):
        train = [i for i in range(n) if k == K or not (lo[k] <= key[i] < hi[k])]
        e = 0
        for a in range(nc + 1):
            for b in range(a + 1):
                exact = sum((fu[i][a] * fu[i][b] for i in train), Fraction(0))
                got = g[k, e]
                assert abs(Fraction(got) - exact) <= Fraction(np.spacing(abs(float(exact)))), (k, a, b, got, float(exact))
                e += 1


def test_fold_gram_rejects_non_finite_data():
    y = np.array([1.0, np.inf, 2.0])
    with pytest.raises(pcv.InvalidInput):
        pcv.fold_gram(y, np.ones((3, 1)), np.arange(3), np.arange(3), np.arange(3) + 1)


def test_bench_reference_arm_line():
    """bench.py --impl reference (the driver's reference arm) prints one JSON line with the
    contract keys; it runs the compiled reference engine (or the oracle port) on host cores only."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["impl"] == "reference" and line["metric"] == "chain-steps/sec" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


def test_benchmark_regroups_sub_blocks_like_presummed_blocks():
    """Early stop keeps one shuffle sub-block per check interval and regroups the completed ones
    into `blocks` benchmark blocks (block g = sub-blocks [g c / B, (g + 1) c / B)). The
    positional host benchmark on c sub-blocks regrouped into B must equal the benchmark on the
    B presummed blocks bit for bit (same summation order), including uneven groups."""
    rng = np.random.default_rng(8)
    nm, nfold, L, stride = 2, 9, 4, 12
    y = rng.standard_normal((nm, nfold, L, stride))
    y2 = y ** 2 + rng.uniform(size=y.shape)
    for sub, B in ((10, 5), (7, 5), (12, 3), (5, 5)):
        starts = [g * sub // B for g in range(B + 1)]
        gy = np.zeros((nm, nfold, L, B))
        gy2 = np.zeros_like(gy)
        for g in range(B):
            for d in range(starts[g], starts[g + 1]):
                gy[..., g] += y[..., d]
                gy2[..., g] += y2[..., d]
        a, ah = pcv.benchmark_host(nm, nfold, L, stride, sub, 200, 7, 50, y.ravel(), y2.ravel(), block_groups=B)
        b, bh = pcv.benchmark_host(nm, nfold, L, B, B, 200, 7, 50, gy.ravel(), gy2.ravel())
        np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(ah, bh)

"""GPU tests of the device accumulators (closed forms and online = two-pass, the reference's
test_scoring.cpp / test_accum.cpp cases), of the engine's input validation (errors.hpp taxonomy
through the C ABI) and of the stepwise / early-stop driver."""
import numpy as np
import pytest

from paper_2310_07002_b200 import abi, pcv
from parity_util import Case
from test_oracle_pinning import score_streams as oracle_streams, two_pass

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = pcv.Context(0)
    yield c
    c.close()


def test_device_logs_closed_cases(ctx):  # test_scoring.cpp:12-42
    logc = np.log(0.37)
    out = ctx.score_streams(np.full((2, 100), logc), center=logc, batch=10, blocks=5)
    assert abs(out["estimate"] - logc) < 1e-12 * abs(logc) and abs(out["mc"]) < 1e-12
    out = ctx.score_streams([[np.log(0.5), np.log(1.5)]], center=0.0, batch=1, blocks=1)
    assert abs(out["estimate"]) < 1e-14
    out = ctx.score_streams(np.full((1, 20), -np.inf), batch=5, blocks=2)
    assert out["estimate"] == -np.inf and out["fault"] == 1 and np.isinf(out["mc"])
    # faults: NaN / +inf draws are counted and fed as zero density (accum.cpp:165-176)
    s = np.full((2, 50), -1.0)
    s[0, 3] = np.nan
    s[1, 7] = np.inf
    out = ctx.score_streams(s, batch=10, blocks=5)
    assert out["fault"] == 1 and np.isfinite(out["estimate"])


def test_device_online_equals_two_pass_and_oracle(ctx):  # test_accum.cpp:180-202, acceptance C1
    rng = np.random.default_rng(2)
    for trial in range(10):
        ch = -2.0 + 0.8 * rng.standard_normal((4, 900))
        out = ctx.score_streams(ch, center=-2.0, batch=50, blocks=5)
        ref_score, ref_naive, ref_mc = two_pass(ch, 50)
        assert abs(out["estimate"] - ref_score) <= 1e-10 * abs(ref_score)
        assert abs(out["naive"] - ref_naive) <= 1e-8 * ref_naive
        assert abs(out["mc"] - ref_mc) <= 1e-8 * ref_mc
        o = oracle_streams(ch, -2.0, 50, 5)
        assert abs(out["rhat"] - o[5]) <= 1e-12 * o[5] and out["batches"] == o[6]


def test_rhat_closed_form_on_device(ctx):  # test_diagnostics.cpp:21-29: chains {1,2},{3,4}
    out = ctx.score_streams(np.log([[1.0, 2.0], [3.0, 4.0]]), center=0.0, batch=1, blocks=1)
    # R-hat is computed on the log-scores s - C: sums of log 1, log 2 / log 3, log 4
    s = np.log([[1.0, 2.0], [3.0, 4.0]])
    n, l = 2, 2
    w = np.mean([np.var(c, ddof=1) for c in s])
    b = n * np.var(s.mean(axis=1), ddof=1)
    assert abs(out["rhat"] - np.sqrt(((n - 1) / n * w + b / n) / w)) < 1e-12


def _ctx_with(name):
    case = Case(name)
    c = pcv.Context(0)
    for i, (m, kp, bank) in enumerate(zip(case.models, case.kparams, case.banks)):
        c.add_model(m, kp, bank, model_id=i)
    return case, c


def test_run_config_validation():  # RunConfig::validate, engine.cpp:21-30; run_pcv 258-271
    case, c = _ctx_with("cfg1_linreg_loo")
    bad = [dict(chains=1), dict(iters=0), dict(warmup=-1), dict(iters=10, batch_size=50), dict(blocks=0),
           dict(bench_draws=0), dict(checkpoint_every=-1)]
    for kw in bad:
        base = dict(chains=4, iters=100, warmup=10, batch_size=10, bench_draws=10)
        base.update(kw)
        with pytest.raises(pcv.InvalidInput):
            c.run(abi.run_config(**base))
    with pytest.raises(pcv.InvalidInput):
        c.run(abi.run_config(chains=4, iters=100, warmup=10, batch_size=10, score=7))
    c.close()


def test_model_validation():
    case = Case("cfg1_linreg_loo")
    with pcv.Context(0) as c:
        with pytest.raises(pcv.InvalidInput):  # empty bank
            c.add_model(case.models[0], case.kparams[0], np.zeros((0, 9)))
        bad_mass = pcv.KernelParams(0.1, 32, -np.ones(9))
        with pytest.raises(pcv.InvalidInput):
            c.add_model(case.models[0], bad_mass, case.banks[0])
        d = case.data
        f = pcv.FoldAssignment(3, np.zeros(d.n_obs, np.int32))  # folds 1, 2 empty
        with pytest.raises(pcv.InvalidInput):
            c.add_model(pcv.GroupedRegressionModel("M", d, f), case.kparams[0], case.banks[0])


def test_stepwise_equals_single_call():
    """begin/advance/fold_stats + merge (the sharded driver) == pcvg_run on one device, bitwise."""
    case, c = _ctx_with("ex1_grouped_logo")
    cfg = abi.run_config(chains=4, iters=60, warmup=10, batch_size=10, bench_draws=20, seed=3)
    rep = c.run(cfg)
    c.begin(cfg)
    c.advance(25)
    c.advance(35)
    cols, divs, dropped, done = c.fold_stats(case.K)
    yx, yx2 = c.block_sums(case.K, 5)
    rep2 = pcv.merge(2, case.K, cfg, done, True, cols, yx, yx2)
    for k in ("delta_hat", "mcse", "epistemic_se", "rhat_max", "prob_a_better"):
        assert rep[k] == rep2[k], k
    np.testing.assert_array_equal(rep["benchmark"], rep2["benchmark"])
    assert np.array_equal(rep["divergences"], divs) and rep["dropped_batch_draws"] == dropped
    c.close()


def test_fold_shards_are_independent():
    """A fold range run alone gives the same per-fold results as inside the full run (chains are
    keyed by global (model, fold, chain): GPU-count invariance)."""
    case, c = _ctx_with("cfg1_linreg_loo")
    cfg = abi.run_config(chains=4, iters=40, warmup=10, batch_size=10, bench_draws=5, seed=2)
    c.begin(cfg)
    c.advance(40)
    full, _, _, _ = c.fold_stats(case.K)
    cfg2 = abi.run_config(chains=4, iters=40, warmup=10, batch_size=10, bench_draws=5, seed=2,
                          fold_begin=30, fold_end=55)
    c.begin(cfg2)
    c.advance(40)
    part, _, _, _ = c.fold_stats(25)
    for k in ("estimate", "mc_contribution", "rhat"):
        np.testing.assert_array_equal(part[k], full[k][30:55])
    c.close()


def test_early_stop_rule():
    case, c = _ctx_with("ex1_grouped_logo")
    cfg = abi.run_config(chains=4, iters=400, warmup=20, batch_size=10, bench_draws=100,
                         checkpoint_every=50, early_stop=1, seed=1)
    rep = c.run(cfg)
    assert rep["iters_run"] <= 400 and rep["iters_run"] % 50 == 0
    assert rep["n_checkpoints"] == rep["iters_run"] // 50
    if rep["iters_run"] < 400:
        assert rep["mcse"] < rep["epistemic_se"] and rep["verdict_pass"] == 1
    c.close()


def test_device_benchmark_equals_host_sequential():
    """bench_kernel (positional Philox stream per item) == the reference's sequential shuffle
    benchmark (diagnostics.cpp:76-101) on the same block sums, with failed folds excluded and
    with fewer blocks used than stored (early-stop probe)."""
    case, c = _ctx_with("ex1_grouped_logo")
    cfg = abi.run_config(chains=4, iters=60, warmup=10, batch_size=10, bench_draws=64, seed=5)
    c.begin(cfg)
    c.advance(60)
    cols, divs, dropped, done = c.fold_stats(case.K)
    yx, yx2 = c.block_sums(case.K, 5)
    failed = np.zeros(case.K, np.int32)
    failed[[2, 7, 31]] = 1
    for blocks_used in (5, 3):
        mx, nh = c.benchmark(failed, 0, int(np.sum(failed == 0)), blocks_used)
        assert nh.max() == 0
        hx, hh = pcv.benchmark_host(2, case.K, 4, 5, blocks_used, done, cfg.seed, cfg.bench_draws, yx, yx2, failed)
        np.testing.assert_array_equal(mx, hx)
    cols["failed"] = np.tile(failed, 2)
    seq = pcv.merge(2, case.K, cfg, done, True, cols, yx, yx2)
    mx, _ = c.benchmark(failed, 0, int(np.sum(failed == 0)), 5)
    dev = pcv.merge_bench(2, case.K, cfg, done, True, cols, mx)
    np.testing.assert_array_equal(dev["benchmark"], seq["benchmark"])
    c.close()


def test_shared_streams_identical_models_give_zero_delta():
    """test_engine.cpp:187-201: two identical models with shared_streams consume the same chain
    streams (engine.cpp:299-300), so every fold difference is exactly zero."""
    case = Case("ex1_grouped_logo")
    c = pcv.Context(0)
    m, kp, bank = case.models[0], case.kparams[0], case.banks[0]
    c.add_model(m, kp, bank, model_id=0)
    c.add_model(m, kp, bank, model_id=1)
    rep = c.run(abi.run_config(chains=4, iters=40, warmup=10, batch_size=10, bench_draws=10, seed=2,
                               shared_streams=1))
    assert np.all(rep["delta_k"] == 0.0) and rep["delta_hat"] == 0.0
    rep2 = c.run(abi.run_config(chains=4, iters=40, warmup=10, batch_size=10, bench_draws=10, seed=2))
    assert np.any(rep2["delta_k"] != 0.0)  # independent streams otherwise
    c.close()


def test_sharded_driver_single_rank_equals_run():
    """dist.run_pcv_sharded (fold-sharded multi-GPU driver: per-checkpoint table gathers, device
    benchmark at global stream offsets, MAX reduction) in a one-rank process group reproduces
    pcvg_run bit for bit."""
    import os
    import socket
    import torch.distributed as tdist
    from paper_2310_07002_b200 import dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=0, world_size=1)
    try:
        case = Case("ex1_grouped_logo")
        inputs = [pcv.ModelInput(m, pcv.FullDataFit(kp, b), i)
                  for i, (m, kp, b) in enumerate(zip(case.models, case.kparams, case.banks))]
        cfg = abi.run_config(chains=4, iters=60, warmup=10, batch_size=10, bench_draws=30, seed=4,
                             checkpoint_every=30)
        rep = pcv.run_pcv(inputs, cfg)
        rep2 = dist.run_pcv_sharded(inputs, cfg, device=0)
        for k in ("delta_hat", "mcse", "epistemic_se", "rhat_max", "prob_a_better", "verdict_quantile_value"):
            assert rep[k] == rep2[k], k
        for k in ("estimate", "rhat", "failed", "divergences", "benchmark"):
            np.testing.assert_array_equal(rep[k], rep2[k])
        np.testing.assert_array_equal(rep["snapshots"], rep2["snapshots"])
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("name", ["cfg1_linreg_loo", "seasonal_timeblocks", "seasonal_hvblock"])
def test_lean_kernel_matches_general_kernel(name):
    """The lean all-global sufficient-statistics kernel (lean_kernel.cu: warm-up and sampling of
    J = 1 grouped regression and seasonal AR) against the general sufficient-statistics kernel it
    replaces on those launches (PCVG_NO_LEAN): the same arithmetic on the same streams, so a short
    run's per-fold estimates and R-hat agree to rounding on (nearly) every fold."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path[:0] = ["tests", "tests/golden", "."]
from parity_util import Case
from paper_2310_07002_b200 import abi, pcv
case = Case(sys.argv[2])
with pcv.Context(0) as c:
    for i, (m, kp, bank) in enumerate(zip(case.models, case.kparams, case.banks)):
        c.add_model(m, kp, bank, model_id=i)
    rep = c.run(abi.run_config(chains=4, iters=16, warmup=4, batch_size=4, blocks=4, bench_draws=10, seed=9))
np.save(sys.argv[1], np.stack([rep["estimate"], rep["rhat"]]))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for tag, env in (("lean", {}), ("general", {"PCVG_NO_LEAN": "1"})):
        path = f"/tmp/pcvg_lean_{tag}_{name}.npy"
        r = subprocess.run([sys.executable, "-c", code, path, name], env={**os.environ, **env}, capture_output=True,
                           text=True, timeout=600, cwd=root)
        assert r.returncode == 0, r.stderr
        out[tag] = np.load(path)
    a, b = out["lean"], out["general"]
    ok = np.isfinite(b)
    np.testing.assert_array_equal(ok, np.isfinite(a))
    rel = np.abs(a[ok] - b[ok]) / (1.0 + np.abs(b[ok]))
    assert np.mean(rel <= 1e-10) >= 0.95, np.sort(rel)[-5:]

"""Multi-process (world_size 2, gloo, CPU) test of the fold-sharded path: each rank owns a
contiguous fold range, the per-fold tables and block sums are all-gathered in rank order, and the
merged Step-4 statistics are bit-identical to the single-process merge (the reference's
thread-count invariance, test_engine.cpp:135-147, as GPU-count invariance)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2310_07002_b200 import abi, dist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _tables(n_models, K, L, D, seed=0):
    rng = np.random.default_rng(seed)
    cols = {}
    for name, dt in abi.FOLD_COLUMNS:
        if dt is np.float64:
            cols[name] = rng.standard_normal(n_models * K) * (0.1 if name != "estimate" else 3.0)
        else:
            cols[name] = np.zeros(n_models * K, dtype=dt)
    cols["mc_contribution"] = np.abs(cols["mc_contribution"])
    cols["naive_contribution"] = np.abs(cols["naive_contribution"])
    cols["rhat"] = 1.0 + np.abs(cols["rhat"])
    for k in (3, 20):  # failed folds (both models): excluded from the benchmark stream
        cols["failed"][k] = cols["failed"][K + k] = 1
    y_x = rng.standard_normal(n_models * K * L * D)
    y_x2 = y_x ** 2 + np.abs(rng.standard_normal(y_x.shape))
    return cols, y_x, y_x2


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as tdist
    from paper_2310_07002_b200 import pcv
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    n_models, K, L, D = 2, 37, 4, 5
    cols, y_x, y_x2 = _tables(n_models, K, L, D)
    fb, fe = dist.shard_range(K, rank, world)
    # this rank's shard, model-major like pcvg_fold_stats writes it
    mine = {k: np.concatenate([v[m * K + fb:m * K + fe] for m in range(n_models)]) for k, v in cols.items()}
    yxm = np.concatenate([y_x[(m * K + fb) * L * D:(m * K + fe) * L * D] for m in range(n_models)])
    yx2m = np.concatenate([y_x2[(m * K + fb) * L * D:(m * K + fe) * L * D] for m in range(n_models)])
    full = dist.gather_fold_tables(mine, n_models)
    g_yx = dist.gather_rows(yxm, n_models)
    g_yx2 = dist.gather_rows(yx2m, n_models)
    cfg = abi.run_config(chains=L, iters=100, batch_size=10, blocks=D, bench_draws=50)
    rep = pcv.merge(n_models, K, cfg, 100, True, full, g_yx, g_yx2)
    # sharded benchmark: each rank consumes its own items at their global stream positions
    # (pcvg_benchmark's arithmetic on host block sums), then MAX across ranks
    failed_local = cols["failed"][fb:fe]
    before, total = dist.shard_benchmark_offsets(failed_local)
    mx, nh = pcv.benchmark_host(n_models, fe - fb, L, D, D, 100, cfg.seed, cfg.bench_draws, yxm, yx2m,
                                failed_local, before, total)
    mx, nh = dist.reduce_benchmark(mx, nh)
    rep2 = pcv.merge_bench(n_models, K, cfg, 100, True, full, mx)
    out_q.put((rank, rep["delta_hat"], rep["mcse"], rep["epistemic_se"], rep["rhat_max"],
               rep["benchmark"].tolist(), {k: v.tolist() for k, v in full.items()},
               rep2["benchmark"].tolist(), int(nh.max())))
    tdist.destroy_process_group()


def test_sharded_merge_is_gpu_count_invariant():
    from paper_2310_07002_b200 import pcv
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n_models, K, L, D = 2, 37, 4, 5
    cols, y_x, y_x2 = _tables(n_models, K, L, D)
    cfg = abi.run_config(chains=L, iters=100, batch_size=10, blocks=D, bench_draws=50)
    single = pcv.merge(n_models, K, cfg, 100, True, cols, y_x, y_x2)
    for rank, dh, mcse, ese, rmax, bench, full, bench2, rejected in results:
        assert rejected == 0
        assert np.array_equal(np.asarray(bench2), single["benchmark"])  # sharded == sequential
        for k, v in cols.items():
            assert np.array_equal(np.asarray(full[k], dtype=v.dtype), v), k
        assert dh == single["delta_hat"] and mcse == single["mcse"] and ese == single["epistemic_se"]
        assert rmax == single["rhat_max"]
        assert np.array_equal(np.asarray(bench), single["benchmark"])


def test_shard_ranges_partition():
    for K in (1, 7, 100, 10000):
        for world in (1, 2, 3, 8):
            r = [dist.shard_range(K, i, world) for i in range(world)]
            assert r[0][0] == 0 and r[-1][1] == K
            assert all(r[i][1] == r[i + 1][0] for i in range(world - 1))


def test_positional_benchmark_equals_sequential():
    """pcvg_benchmark's positional stream == the reference's sequential below() stream
    (diagnostics.cpp:82-98) on one shard, with failed folds and fewer blocks used than stored."""
    from paper_2310_07002_b200 import pcv
    n_models, K, L, D = 2, 23, 6, 5
    cols, y_x, y_x2 = _tables(n_models, K, L, D, seed=3)
    cfg = abi.run_config(chains=L, iters=80, batch_size=10, blocks=D, bench_draws=40, seed=9)
    single = pcv.merge(n_models, K, cfg, 80, True, cols, y_x, y_x2)
    failed = cols["failed"][:K]
    mx, nh = pcv.benchmark_host(n_models, K, L, D, D, 80, cfg.seed, cfg.bench_draws, y_x, y_x2, failed)
    assert nh.max() == 0
    rep = pcv.merge_bench(n_models, K, cfg, 80, True, cols, mx)
    assert np.array_equal(rep["benchmark"], single["benchmark"])
    assert rep["verdict_quantile_value"] == single["verdict_quantile_value"]

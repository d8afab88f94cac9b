"""Fold sharding across GPUs (one process per GPU, torch.distributed over NCCL; gloo on CPU).

SURVEY.md 8(e): each rank owns a contiguous fold range with all L chains of a fold, so per-fold
R-hat/ESS/LogS need no communication. The only exchange is at check intervals: the per-fold
tables (a few doubles per fold) are all-gathered in rank order = reference fold order (tensor
all-gathers: device buffers over NCCL, host buffers over gloo), and every
rank merges them with pcvg_merge (engine.cpp:117-253) in fold order, so the merge itself is
independent of the GPU count (the reference's thread-count invariance, test_engine.cpp:135-147).
The per-fold inputs are bit-identical for any GPU count wherever a chain's arithmetic does not
depend on the launch geometry: the sufficient-statistics, group-batched and row-split Gaussian
kernels (one chain per thread / lane group). The tensor-core GLM kernels (logistic; Gaussian models
under the ROWS policy) run a shard's last partial wave of 64-chain tiles as row-split clusters whose
partial sums are combined in a different order, and which tiles form that tail depends on the shard
size: those chains agree with a single-GPU run to rounding (~1e-14 relative per gradient), then
diverge chaotically as any two MCMC runs with last-ulp differences do; the estimates agree within
Monte Carlo error (tests/test_gpu_dist.py).
"""
from __future__ import annotations

import numpy as np

from . import abi


def shard_range(K: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous fold range [begin, end) of `rank` (balanced, in fold order)."""
    return rank * K // world, (rank + 1) * K // world


def _coll_device(group=None):
    """Device of the collective buffers: the rank's current CUDA device under NCCL, else the CPU
    (gloo)."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _all_gather_rows(arr: np.ndarray, group=None) -> list:
    """All-gathers a float64 array of n_rank rows (n_rank may differ by rank) with tensor
    collectives: the row counts first, then the rows padded to the largest count. Returns the
    per-rank arrays in rank order (NCCL moves device buffers over NVLink; gloo host buffers)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = _coll_device(group)
    a = np.ascontiguousarray(arr, dtype=np.float64)
    tail = a.shape[1:]
    n = torch.tensor([a.shape[0]], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    rows = max(counts)
    buf = torch.zeros((rows,) + tail, dtype=torch.float64, device=dev)
    if a.shape[0]:
        buf[:a.shape[0]] = torch.from_numpy(a).to(dev)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return [p[:c].cpu().numpy() for p, c in zip(parts, counts)]


def gather_fold_tables(cols: dict, n_models: int, group=None) -> dict:
    """All-gathers per-shard fold tables (model-major rows within each shard) into full tables in
    model-major, fold order: one [rows x columns] float64 all-gather (every column is a double or
    an integer far below 2^53, so the round trip is exact)."""
    names = [name for name, _ in abi.FOLD_COLUMNS]
    mine = np.stack([np.asarray(cols[name], dtype=np.float64) for name in names], axis=1)
    parts = _all_gather_rows(mine, group)
    out = {}
    for j, name in enumerate(names):
        dtype = np.asarray(cols[name]).dtype
        per_model = []
        for m in range(n_models):
            for p in parts:
                nf = p.shape[0] // n_models
                per_model.append(p[m * nf:(m + 1) * nf, j])
        out[name] = np.concatenate(per_model).astype(dtype)
    return out


def gather_rows(arr: np.ndarray, n_models: int, group=None) -> np.ndarray:
    """Same gather for per-chain / per-block arrays laid out model-major per shard."""
    a = np.asarray(arr)
    parts = _all_gather_rows(a, group)
    per_model = []
    for m in range(n_models):
        for p in parts:
            n = p.shape[0] // n_models
            per_model.append(p[m * n:(m + 1) * n])
    return np.concatenate(per_model).astype(a.dtype)


def shard_benchmark_offsets(failed_local, group=None) -> tuple[int, int]:
    """(non-failed folds before this shard, non-failed folds in total) from an all-gather of the
    per-shard non-failed counts: the global stream position of this shard's benchmark items
    (pcvg_benchmark, diagnostics.cpp:82-98)."""
    import torch.distributed as dist

    mine = int(np.sum(np.asarray(failed_local) == 0)) if failed_local is not None else 0
    parts = _all_gather_rows(np.array([mine], dtype=np.float64), group)
    counts = [int(p[0]) for p in parts]
    rank = dist.get_rank(group)
    return int(sum(counts[:rank])), int(sum(counts))


def reduce_benchmark(rep_max: np.ndarray, needs_host: np.ndarray, device=None, group=None):
    """All-reduce MAX of the per-shard replicate maxima and of the rejection flags."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.concatenate([rep_max, needs_host.astype(np.float64)]))
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    t = t.cpu().numpy()
    R = rep_max.shape[0]
    return t[:R].copy(), t[R:].astype(np.int32)


def failed_from_divergences(div: np.ndarray, n_models: int, K: int, L: int, iters: int) -> np.ndarray:
    """Failed folds (engine.cpp:385-397): every chain of some model divergent on > N/2 iterations."""
    d = div.reshape(n_models, K, L)
    bad = np.all(d * 2 > iters, axis=2)  # [m, k]
    f = np.any(bad, axis=0).astype(np.int32)
    return np.tile(f, n_models)


def run_pcv_sharded(inputs, cfg, device=0, group=None):
    """run_pcv (engine.cpp:257-483) with the folds sharded across the ranks of `group` (one
    process per GPU): every rank samples its contiguous fold range on its own device; at each
    checkpoint the per-fold tables are all-gathered in fold order and merged identically on every
    rank; the shuffle benchmark runs on each rank's own block sums at its global stream offset and
    the replicate maxima are MAX-reduced. No block sums or chain states leave their GPU. Returns
    the report dict (pcv.Context.run's layout) on every rank."""
    import copy

    import torch.distributed as dist

    from . import pcv

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    K = inputs[0].model.K
    nm = len(inputs)
    fb, fe = shard_range(K, rank, world)
    cfg_s = copy.copy(cfg)
    cfg_s.fold_begin, cfg_s.fold_end = fb, fe
    if fe == fb:
        raise pcv.InvalidInput("more ranks than folds")
    checkpoints = list(range(cfg.checkpoint_every, cfg.iters, cfg.checkpoint_every)) if cfg.checkpoint_every > 0 else []
    checkpoints.append(cfg.iters)
    # shuffle sub-blocks stored per chain (one per check interval under early stop)
    d_stride = cfg.iters // cfg.checkpoint_every if cfg.early_stop else cfg.blocks
    snaps = []
    dev = None
    try:
        import torch
        if torch.cuda.is_available() and dist.get_backend(group) == "nccl":
            dev = torch.device("cuda", device)
    except Exception:
        dev = None

    def shard_benchmark(failed_local, sub_used):
        if failed_local is None:
            failed_local = np.zeros(fe - fb, dtype=np.int32)
        before, total = shard_benchmark_offsets(failed_local, group)
        mx, nh = ctx.benchmark(failed_local, before, total, sub_used)
        return reduce_benchmark(mx, nh, dev, group)

    with pcv.Context(device) as ctx:
        for mi in inputs:
            ctx.add_model(mi.model, mi.fit.kparams, mi.fit.draws, mi.model_id)
        ctx.begin(cfg_s)
        done = 0
        for ci, t in enumerate(checkpoints):
            ctx.advance(t - done)
            done = t
            cols, div, dropped, iters = ctx.fold_stats(fe - fb)
            full = gather_fold_tables(cols, nm, group)
            sub_used = iters // cfg.checkpoint_every if cfg.early_stop else cfg.blocks
            last = ci + 1 == len(checkpoints)
            final = last
            if cfg.early_stop and not last and sub_used >= cfg.blocks:
                # the early-stop probe of pcvg_run: no exclusions, benchmark over every fold
                part = dict(full)
                part["failed"] = np.zeros_like(part["failed"])
                mx, nh = shard_benchmark(None, sub_used)
                if nh.max() > 0:
                    yx, yx2 = ctx.block_sums(fe - fb, d_stride)
                    probe = pcv.merge(nm, K, cfg, iters, 2, part, gather_rows(yx, nm, group),
                                      gather_rows(yx2, nm, group))
                else:
                    probe = pcv.merge_bench(nm, K, cfg, iters, 2, part, mx)
                final = bool(probe["verdict_pass"]) and probe["benchmark_count"] > 0 and \
                    np.isfinite(probe["rhat_max"]) and probe["mcse"] < probe["epistemic_se"]
            if not final:
                part = dict(full)
                part["failed"] = np.zeros_like(part["failed"])
                rep = pcv.merge(nm, K, cfg, iters, False, part)
            else:
                failed_local = cols["failed"][: fe - fb]
                mx, nh = shard_benchmark(failed_local, sub_used)
                if nh.max() > 0:  # a below() rejection: the sequential stream needs all block sums
                    yx, yx2 = ctx.block_sums(fe - fb, d_stride)
                    rep = pcv.merge(nm, K, cfg, iters, True, full, gather_rows(yx, nm, group),
                                    gather_rows(yx2, nm, group))
                else:
                    rep = pcv.merge_bench(nm, K, cfg, iters, True, full, mx)
                for name, _ in abi.FOLD_COLUMNS:  # per-fold columns (merge writes only `failed`)
                    if name != "failed":
                        rep[name] = full[name]
                rep["divergences"] = gather_rows(div, nm, group)
                parts = _all_gather_rows(np.array([float(dropped)]), group)
                rep["dropped_batch_draws"] = int(sum(int(p[0]) for p in parts))
                rep["iters_run"] = iters
            snaps.append([iters, rep["delta_hat"], rep["mcse"], rep["epistemic_se"], rep["prob_a_better"],
                          rep["ess_overall"], rep["rhat_max"]])
            if final:
                break
    rep["snapshots"] = np.array(snaps)
    rep["n_checkpoints"] = len(snaps)
    return rep

"""Fold sharding across GPUs (one process per GPU, torch.distributed over NCCL; gloo on CPU).

SURVEY.md 8(e): each rank owns a contiguous fold range with all L chains of a fold, so per-fold
R-hat/ESS/LogS need no communication. The only exchange is at check intervals: the per-fold
tables (a few doubles per fold) are all-gathered in rank order = reference fold order, and every
rank merges them with pcvg_merge (engine.cpp:117-253). Because the merge sums in fold order, the
headline statistics are bit-identical for any GPU count (the reference's thread-count invariance,
test_engine.cpp:135-147, becomes GPU-count invariance).
"""
from __future__ import annotations

import numpy as np

from . import abi


def shard_range(K: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous fold range [begin, end) of `rank` (balanced, in fold order)."""
    return rank * K // world, (rank + 1) * K // world


def gather_fold_tables(cols: dict, n_models: int, group=None) -> dict:
    """All-gathers per-shard fold tables (model-major rows within each shard) into full tables in
    model-major, fold order. Uses all_gather_object so it runs on NCCL and gloo alike."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    parts = [None] * world
    dist.all_gather_object(parts, {k: np.asarray(v) for k, v in cols.items()}, group=group)
    out = {}
    for name, _ in abi.FOLD_COLUMNS:
        per_model = []
        for m in range(n_models):
            chunks = []
            for p in parts:
                arr = p[name]
                nf = arr.shape[0] // n_models
                chunks.append(arr[m * nf:(m + 1) * nf])
            per_model.append(np.concatenate(chunks))
        out[name] = np.concatenate(per_model)
    return out


def gather_rows(arr: np.ndarray, n_models: int, group=None) -> np.ndarray:
    """Same gather for per-chain / per-block arrays laid out model-major per shard."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    parts = [None] * world
    dist.all_gather_object(parts, np.asarray(arr), group=group)
    per_model = []
    for m in range(n_models):
        for p in parts:
            n = p.shape[0] // n_models
            per_model.append(p[m * n:(m + 1) * n])
    return np.concatenate(per_model)


def failed_from_divergences(div: np.ndarray, n_models: int, K: int, L: int, iters: int) -> np.ndarray:
    """Failed folds (engine.cpp:385-397): every chain of some model divergent on > N/2 iterations."""
    d = div.reshape(n_models, K, L)
    bad = np.all(d * 2 > iters, axis=2)  # [m, k]
    f = np.any(bad, axis=0).astype(np.int32)
    return np.tile(f, n_models)

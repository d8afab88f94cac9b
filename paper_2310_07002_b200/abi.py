"""ctypes mirror of include/pcvg.h (the C ABI of libpcvg.so).

Plain data structs only; the same layouts are consumed by the product library and, in the
tests, by the CPU oracle (oracle/pcv_oracle.c) and the reference shim (oracle/ref_shim.cpp).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ABI_VERSION = 3

OK, INVALID_INPUT, NUMERIC_FAULT, ADAPTATION_FAILURE, UNDEFINED_DIAGNOSTIC, \
    UNSUPPORTED_SCORE, CUDA_ERROR, COMM_ERROR = range(8)

FAMILY_GROUPED, FAMILY_RADON, FAMILY_SEASONAL_AR, FAMILY_LOGISTIC, FAMILY_RAT_GROWTH = range(5)
SCORE_LOGS, SCORE_HS, SCORE_DSS = range(3)
RHO_HALF_OPEN, RHO_SYMMETRIC = range(2)
STREAM_CHAIN_SAMPLING, STREAM_CHAIN_INIT, STREAM_FULL_DATA, STREAM_SIMULATE, STREAM_KFOLD, \
    STREAM_BENCHMARK, STREAM_STEP_INIT = range(1, 8)

P_f64 = C.POINTER(C.c_double)
P_i32 = C.POINTER(C.c_int32)
P_i64 = C.POINTER(C.c_int64)
P_u64 = C.POINTER(C.c_uint64)


class Dataset(C.Structure):
    _fields_ = [("n_obs", C.c_int64), ("n_cov", C.c_int32), ("y", P_f64), ("x", P_f64),
                ("group_id", P_i32), ("time_index", P_i64)]


class Folds(C.Structure):
    _fields_ = [("K", C.c_int32), ("test_index", P_i32), ("intervals", P_i64)]


class ModelSpec(C.Structure):
    _fields_ = [("family", C.c_int32), ("covariate_mask", P_i32), ("include_floor", C.c_int32),
                ("ar_order", C.c_int32), ("dummies", C.c_int32), ("rho_transform", C.c_int32),
                ("per_subject_slope", C.c_int32)]


class Kernel(C.Structure):
    _fields_ = [("step_size", C.c_double), ("n_leapfrog", C.c_int32), ("inv_mass_diag", P_f64)]


class RunConfig(C.Structure):
    _fields_ = [("chains", C.c_int32), ("iters", C.c_int64), ("warmup", C.c_int64),
                ("batch_size", C.c_int32), ("blocks", C.c_int32), ("bench_draws", C.c_int32),
                ("bench_quantile", C.c_double), ("seed", C.c_uint64), ("score", C.c_int32),
                ("checkpoint_every", C.c_int64), ("shared_streams", C.c_int32),
                ("fold_begin", C.c_int32), ("fold_end", C.c_int32), ("early_stop", C.c_int32)]


class FoldTable(C.Structure):
    _fields_ = [("estimate", P_f64), ("log_f_hat", P_f64), ("mc_contribution", P_f64),
                ("naive_contribution", P_f64), ("ess", P_f64), ("rhat", P_f64),
                ("batches", P_i64), ("fault", P_i32), ("failed", P_i32), ("dss_ridged", P_i32)]


class Report(C.Structure):
    _fields_ = [("folds", FoldTable), ("divergences", P_i64), ("delta_k", P_f64),
                ("snapshots", P_f64), ("benchmark", P_f64),
                ("delta_hat", C.c_double), ("mcse", C.c_double), ("sigma2_delta", C.c_double),
                ("epistemic_se", C.c_double), ("prob_a_better", C.c_double),
                ("ess_overall", C.c_double), ("rhat_max", C.c_double),
                ("score_total", C.c_double * 2), ("numeric_faults", C.c_int64 * 2),
                ("rhat_excluded", C.c_int32 * 2), ("dropped_batch_draws", C.c_int64),
                ("n_checkpoints", C.c_int32), ("benchmark_count", C.c_int32),
                ("verdict_pass", C.c_int32), ("verdict_quantile", C.c_double),
                ("verdict_quantile_value", C.c_double), ("verdict_observed", C.c_double),
                ("iters_run", C.c_int64), ("warmup_ms", C.c_double), ("sampling_ms", C.c_double),
                ("gpu_launches", C.c_int64)]


class AdaptConfig(C.Structure):
    _fields_ = [("chains", C.c_int32), ("warmup", C.c_int64), ("draws", C.c_int64),
                ("n_leapfrog", C.c_int32), ("target_accept", C.c_double),
                ("init_step_size", C.c_double)]


class Fit(C.Structure):
    _fields_ = [("step_size", C.c_double), ("inv_mass_diag", P_f64), ("draws", P_f64),
                ("rhat", P_f64), ("ess", P_f64), ("step_trace", P_f64),
                ("divergences", C.c_int64), ("mean_accept", C.c_double), ("device_ms", C.c_double)]


def ptr(a, ctype):
    """Pointer into a contiguous numpy array (None passes NULL)."""
    if a is None:
        return C.cast(None, C.POINTER(ctype))
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data_as(C.POINTER(ctype))


FOLD_COLUMNS = [("estimate", np.float64), ("log_f_hat", np.float64),
                ("mc_contribution", np.float64), ("naive_contribution", np.float64),
                ("ess", np.float64), ("rhat", np.float64), ("batches", np.int64),
                ("fault", np.int32), ("failed", np.int32), ("dss_ridged", np.int32)]
_CT = {np.float64: C.c_double, np.int64: C.c_int64, np.int32: C.c_int32}


def new_fold_table(rows):
    """Allocates the numpy columns of a pcvg_fold_table; returns (struct, dict of arrays)."""
    cols = {name: np.zeros(rows, dtype=dt) for name, dt in FOLD_COLUMNS}
    st = FoldTable(**{name: ptr(cols[name], _CT[dt]) for name, dt in FOLD_COLUMNS})
    return st, cols


def checkpoint_count(iters, checkpoint_every):
    """engine.cpp:279-283: checkpoints every `checkpoint_every` below N, always ending at N."""
    if checkpoint_every > 0:
        return len(range(checkpoint_every, iters, checkpoint_every)) + 1
    return 1


def new_report(n_models, K, L, n_ckpt, bench_draws):
    """Allocates a pcvg_report with its numpy arrays; returns (struct, dict of arrays)."""
    ft, cols = new_fold_table(n_models * K)
    arrs = dict(cols)
    arrs["divergences"] = np.zeros(n_models * K * L, dtype=np.int64)
    arrs["delta_k"] = np.zeros(K, dtype=np.float64)
    arrs["snapshots"] = np.zeros(max(n_ckpt, 1) * 7, dtype=np.float64)
    arrs["benchmark"] = np.zeros(max(bench_draws, 1), dtype=np.float64)
    rep = Report(folds=ft, divergences=ptr(arrs["divergences"], C.c_int64),
                 delta_k=ptr(arrs["delta_k"], C.c_double),
                 snapshots=ptr(arrs["snapshots"], C.c_double),
                 benchmark=ptr(arrs["benchmark"], C.c_double))
    return rep, arrs


def report_dict(rep, arrs, n_models):
    out = {k: getattr(rep, k) for k in ("delta_hat", "mcse", "sigma2_delta", "epistemic_se",
                                        "prob_a_better", "ess_overall", "rhat_max",
                                        "dropped_batch_draws", "n_checkpoints",
                                        "benchmark_count", "verdict_pass", "verdict_quantile",
                                        "verdict_quantile_value", "verdict_observed",
                                        "iters_run", "warmup_ms", "sampling_ms",
                                        "gpu_launches")}
    out["score_total"] = [rep.score_total[m] for m in range(n_models)]
    out["numeric_faults"] = [rep.numeric_faults[m] for m in range(n_models)]
    out["rhat_excluded"] = [rep.rhat_excluded[m] for m in range(n_models)]
    out.update({k: v.copy() for k, v in arrs.items()})
    out["snapshots"] = out["snapshots"][: 7 * rep.n_checkpoints].reshape(-1, 7)
    out["benchmark"] = out["benchmark"][: rep.benchmark_count]
    return out


class DatasetArrays:
    """Owns contiguous numpy columns and the pcvg_dataset struct pointing at them."""

    def __init__(self, y, x=None, group_id=None, time_index=None):
        self.y = np.ascontiguousarray(y, dtype=np.float64)
        n = self.y.shape[0]
        if x is None:
            x = np.zeros((n, 0))
        x = np.asarray(x, dtype=np.float64)
        if x.ndim == 1:
            x = x.reshape(n, -1)
        self.x = np.ascontiguousarray(x)
        self.group_id = None if group_id is None else np.ascontiguousarray(group_id, dtype=np.int32)
        self.time_index = None if time_index is None else np.ascontiguousarray(time_index, dtype=np.int64)
        self.struct = Dataset(n_obs=n, n_cov=self.x.shape[1], y=ptr(self.y, C.c_double),
                              x=ptr(self.x if self.x.size else np.zeros(1), C.c_double),
                              group_id=ptr(self.group_id, C.c_int32),
                              time_index=ptr(self.time_index, C.c_int64))

    @property
    def n_obs(self):
        return self.y.shape[0]

    @property
    def n_groups(self):
        return 0 if self.group_id is None else int(self.group_id.max()) + 1


class FoldArrays:
    """A partition (test_index) or hv-block intervals, plus the pcvg_folds struct."""

    def __init__(self, K, test_index=None, intervals=None):
        self.K = int(K)
        self.test_index = None if test_index is None else np.ascontiguousarray(test_index, dtype=np.int32)
        self.intervals = None if intervals is None else np.ascontiguousarray(intervals, dtype=np.int64).reshape(-1)
        self.struct = Folds(K=self.K, test_index=ptr(self.test_index, C.c_int32),
                            intervals=ptr(self.intervals, C.c_int64))


class SpecArrays:
    def __init__(self, family, covariate_mask=None, include_floor=1, ar_order=1, dummies=0,
                 rho_transform=RHO_HALF_OPEN, per_subject_slope=0):
        self.family = family
        self.mask = None if covariate_mask is None else np.ascontiguousarray(covariate_mask, dtype=np.int32)
        self.struct = ModelSpec(family=family, covariate_mask=ptr(self.mask, C.c_int32),
                                include_floor=int(include_floor), ar_order=int(ar_order),
                                dummies=int(dummies), rho_transform=int(rho_transform),
                                per_subject_slope=int(per_subject_slope))


class KernelArrays:
    def __init__(self, step_size, n_leapfrog, inv_mass_diag):
        self.inv_mass = np.ascontiguousarray(inv_mass_diag, dtype=np.float64)
        self.step_size = float(step_size)
        self.n_leapfrog = int(n_leapfrog)
        self.struct = Kernel(step_size=self.step_size, n_leapfrog=self.n_leapfrog,
                             inv_mass_diag=ptr(self.inv_mass, C.c_double))


def run_config(chains=4, iters=1000, warmup=100, batch_size=50, blocks=5, bench_draws=500,
               bench_quantile=0.99, seed=1, score=SCORE_LOGS, checkpoint_every=0,
               shared_streams=0, fold_begin=0, fold_end=0, early_stop=0):
    """pcv::RunConfig defaults (engine.hpp:21-45)."""
    return RunConfig(chains=chains, iters=iters, warmup=warmup, batch_size=batch_size,
                     blocks=blocks, bench_draws=bench_draws, bench_quantile=bench_quantile,
                     seed=seed, score=score, checkpoint_every=checkpoint_every,
                     shared_streams=shared_streams, fold_begin=fold_begin, fold_end=fold_end,
                     early_stop=early_stop)


PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PCVG_LIB_PATH") or os.path.join(PKG_DIR, "lib", "libpcvg.so")  # override: tooling builds

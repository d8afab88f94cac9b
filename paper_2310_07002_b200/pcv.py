"""Python mirror of the reference's PCV interface over libpcvg.so (ctypes).

Names and argument meaning follow the reference headers so parity tests read like the
reference's own tests:
  Dataset (dataset.hpp:11-25), FoldAssignment + make_{loo,logo,kfold,time_block}_scheme
  (folds.hpp:10-27) + make_hv_block_scheme (new), GroupedRegressionModel / RadonStyleModel /
  SeasonalARModel (models/*.hpp) + LogisticModel (new), KernelParams (hmc.hpp:14-18),
  FullDataFit (adapt.hpp:55-62), RunConfig (engine.hpp:21-45), run_pcv (engine.hpp:116).
Errors raise the reference taxonomy (errors.hpp:9-37) as Python exceptions. Everything that
computes runs in libpcvg.so on the GPU; a missing library or device raises - there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import abi

P = C.POINTER


class PcvError(RuntimeError):
    code = -1


class InvalidInput(PcvError, ValueError):
    code = abi.INVALID_INPUT


class NumericFault(PcvError):
    code = abi.NUMERIC_FAULT


class AdaptationFailure(PcvError):
    code = abi.ADAPTATION_FAILURE


class UndefinedDiagnostic(PcvError):
    code = abi.UNDEFINED_DIAGNOSTIC


class UnsupportedScore(PcvError):
    code = abi.UNSUPPORTED_SCORE


class CudaError(PcvError):
    code = abi.CUDA_ERROR


_EXC = {c.code: c for c in (InvalidInput, NumericFault, AdaptationFailure, UndefinedDiagnostic,
                            UnsupportedScore, CudaError)}

_lib = None


def _sig(lib, name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args


def load():
    """Loads the in-tree libpcvg.so (built by __graft_entry__.build()); raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(abi.LIB_PATH):
        raise ImportError(f"{abi.LIB_PATH} missing: run `python -m paper_2310_07002_b200.build`")
    lib = C.CDLL(abi.LIB_PATH)
    i32, i64, u64, f64, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p
    pf, pi32, pi64 = abi.P_f64, abi.P_i32, abi.P_i64
    _sig(lib, "pcvg_abi_version", i32, [])
    _sig(lib, "pcvg_last_error", C.c_char_p, [vp])
    _sig(lib, "pcvg_status_name", C.c_char_p, [i32])
    _sig(lib, "pcvg_stream_key", u64, [u64, u64, u64, u64])
    _sig(lib, "pcvg_rng_sequence", i32, [u64, u64, i32, u64, C.c_char_p, abi.P_u64, i64, pf])
    _sig(lib, "pcvg_make_loo", i32, [i64, pi32, pi32])
    _sig(lib, "pcvg_make_logo", i32, [P(abi.Dataset), pi32, pi32])
    _sig(lib, "pcvg_make_kfold", i32, [i64, i32, u64, pi32])
    _sig(lib, "pcvg_make_time_blocks", i32, [P(abi.Dataset), i32, pi32])
    _sig(lib, "pcvg_make_hv_block", i32, [P(abi.Dataset), i32, i64, pi64])
    _sig(lib, "pcvg_make_hv_racine", i32, [P(abi.Dataset), i64, i64, pi64])
    _sig(lib, "pcvg_simulate_grouped", i32, [i32, i32, i32, f64, u64, pf, pf, pi32])
    _sig(lib, "pcvg_simulate_radon", i32, [i32, i32, u64, pf, pf, pi32])
    _sig(lib, "pcvg_simulate_rat", i32, [i32, u64, pf, pf, pi32])
    _sig(lib, "pcvg_simulate_seasonal", i32, [i64, i32, i32, f64, f64, f64, u64, pf, pf, pi64])
    _sig(lib, "pcvg_simulate_linreg", i32, [i64, i32, u64, pf, pf, pi32])
    _sig(lib, "pcvg_simulate_logistic", i32, [i64, i32, u64, pf, pf])
    _sig(lib, "pcvg_create", i32, [i32, P(vp)])
    _sig(lib, "pcvg_destroy", i32, [vp])
    _sig(lib, "pcvg_add_model", i32, [vp, P(abi.Dataset), P(abi.Folds), P(abi.ModelSpec),
                                      P(abi.Kernel), pf, i64, i32, pi32])
    _sig(lib, "pcvg_model_dim", i32, [vp, i32, pi32])
    _sig(lib, "pcvg_set_kernel_policy", i32, [vp, i32])
    _sig(lib, "pcvg_model_test_size", i32, [vp, i32, i32, pi64])
    _sig(lib, "pcvg_eval", i32, [vp, i32, i64, pi32, pf, pf, pf])
    _sig(lib, "pcvg_eval_pred", i32, [vp, i32, i64, pi32, pf, pf])
    _sig(lib, "pcvg_hmc_probe", i32, [vp, i32, i64, pi32, pf, pf, pf, pf, pf, pf, pi32, pi32])
    _sig(lib, "pcvg_hmc_chain", i32, [vp, i32, i32, i32, u64, pf, i64, pf, pi32])
    _sig(lib, "pcvg_leapfrog", i32, [vp, i32, i64, pi32, pf, pf, pf, pf, pi32])
    _sig(lib, "pcvg_score_streams", i32, [vp, i32, i64, pf, f64, i32, i32, pf])
    _sig(lib, "pcvg_checkpoint_count", i32, [P(abi.RunConfig)])
    _sig(lib, "pcvg_run", i32, [vp, P(abi.RunConfig), P(abi.Report)])
    _sig(lib, "pcvg_begin", i32, [vp, P(abi.RunConfig)])
    _sig(lib, "pcvg_advance", i32, [vp, i64])
    _sig(lib, "pcvg_fold_stats", i32, [vp, P(abi.FoldTable), pi64, pi64, pi64])
    _sig(lib, "pcvg_block_sums", i32, [vp, pf, pf])
    _sig(lib, "pcvg_timing", i32, [vp, pf, pi64])
    _sig(lib, "pcvg_merge", i32, [i32, i32, P(abi.RunConfig), i64, i32, P(abi.FoldTable), pf, pf,
                                  P(abi.Report)])
    _sig(lib, "pcvg_benchmark", i32, [vp, pi32, i64, i64, i32, pf, pi32])
    _sig(lib, "pcvg_run_streams", i32, [vp, i32, pf, pf, P(abi.RunConfig), P(abi.Report)])
    _sig(lib, "pcvg_debug_break_fold", i32, [vp, i32, i32])
    _sig(lib, "pcvg_phase_times", i32, [vp, pf, pf])
    _sig(lib, "pcvg_multi_create", i32, [i32, pi32, P(vp)])
    _sig(lib, "pcvg_multi_destroy", i32, [vp])
    _sig(lib, "pcvg_multi_last_error", C.c_char_p, [vp])
    _sig(lib, "pcvg_multi_add_model", i32, [vp, P(abi.Dataset), P(abi.Folds), P(abi.ModelSpec), P(abi.Kernel),
                                            pf, i64, i32, pi32])
    _sig(lib, "pcvg_multi_set_kernel_policy", i32, [vp, i32])
    _sig(lib, "pcvg_multi_run", i32, [vp, P(abi.RunConfig), P(abi.Report)])
    _sig(lib, "pcvg_benchmark_host", i32, [i32, i32, i32, i32, i32, i32, i64, u64, i32, pf, pf, pi32, i64,
                                           i64, pf, pi32])
    _sig(lib, "pcvg_merge_bench", i32, [i32, i32, P(abi.RunConfig), i64, i32, P(abi.FoldTable), pf,
                                        P(abi.Report)])
    _sig(lib, "pcvg_adapt_full_data", i32, [vp, P(abi.Dataset), P(abi.Folds), P(abi.ModelSpec),
                                            P(abi.AdaptConfig), u64, i32, P(abi.Fit)])
    _sig(lib, "pcvg_initial_draw", i32, [P(abi.Dataset), P(abi.Folds), P(abi.ModelSpec), u64, u64, pf])
    _sig(lib, "pcvg_fold_gram", i32, [i64, i32, pf, pf, pi32, i32, pi32, pi32, pf])
    if lib.pcvg_abi_version() != abi.ABI_VERSION:
        raise ImportError("libpcvg.so ABI version mismatch")
    _lib = lib
    return lib


def _check(rc, ctx=None):
    if rc != abi.OK:
        msg = load().pcvg_last_error(ctx).decode()
        raise _EXC.get(rc, PcvError)(msg)


def _p(a, ct=C.c_double):
    return abi.ptr(a, ct)


# ----------------------------------------------------------------- data + folds (host, exact)
class Dataset(abi.DatasetArrays):
    """pcv::Dataset (dataset.hpp:11-25)."""


@dataclass
class FoldAssignment:
    """pcv::FoldAssignment (folds.hpp:10-20), or hv-block interval folds (new)."""
    K: int
    test_index: np.ndarray | None = None
    intervals: np.ndarray | None = None

    def arrays(self):
        return abi.FoldArrays(self.K, self.test_index, self.intervals)


def make_loo_scheme(data):
    ti = np.zeros(data.n_obs, dtype=np.int32)
    K = C.c_int32()
    _check(load().pcvg_make_loo(data.n_obs, _p(ti, C.c_int32), C.byref(K)))
    return FoldAssignment(K.value, ti)


def make_logo_scheme(data):
    ti = np.zeros(data.n_obs, dtype=np.int32)
    K = C.c_int32()
    _check(load().pcvg_make_logo(C.byref(data.struct), _p(ti, C.c_int32), C.byref(K)))
    return FoldAssignment(K.value, ti)


def make_kfold_scheme(data, K, seed):
    n = data if isinstance(data, int) else data.n_obs
    ti = np.zeros(n, dtype=np.int32)
    _check(load().pcvg_make_kfold(n, K, seed, _p(ti, C.c_int32)))
    return FoldAssignment(K, ti)


def make_time_block_scheme(data, K):
    ti = np.zeros(data.n_obs, dtype=np.int32)
    _check(load().pcvg_make_time_blocks(C.byref(data.struct), K, _p(ti, C.c_int32)))
    return FoldAssignment(K, ti)


def make_hv_block_scheme(data, K, h):
    iv = np.zeros(4 * K, dtype=np.int64)
    _check(load().pcvg_make_hv_block(C.byref(data.struct), K, h, _p(iv, C.c_int64)))
    return FoldAssignment(K, None, iv)


def make_hv_racine_scheme(data, v, h):
    iv = np.zeros(4 * data.n_obs, dtype=np.int64)
    _check(load().pcvg_make_hv_racine(C.byref(data.struct), v, h, _p(iv, C.c_int64)))
    return FoldAssignment(data.n_obs, None, iv)


def stream_key(kind, a=0, b=0, c=0):
    return load().pcvg_stream_key(kind, a, b, c)


def rng_sequence(seed, stream, ops, args=None, skip_block=None):
    ops_b = ops.encode() if isinstance(ops, str) else ops
    n = len(ops_b)
    arg = np.zeros(n, dtype=np.uint64) if args is None else np.ascontiguousarray(args, dtype=np.uint64)
    out = np.zeros(n)
    _check(load().pcvg_rng_sequence(seed, stream, int(skip_block is not None), skip_block or 0, ops_b,
                                    _p(arg, C.c_uint64), n, _p(out)))
    return out


# ----------------------------------------------------------------- simulators
def simulate_grouped_regression(groups=50, per_group=5, covariates=4, min_omitted_beta=0.0, seed=1):
    n = groups * per_group
    y, x, g = np.zeros(n), np.zeros(n * covariates), np.zeros(n, dtype=np.int32)
    _check(load().pcvg_simulate_grouped(groups, per_group, covariates, min_omitted_beta, seed,
                                        _p(y), _p(x), _p(g, C.c_int32)))
    return Dataset(y, x.reshape(n, covariates), g)


def simulate_radon_style(houses, counties, seed):
    y, x, g = np.zeros(houses), np.zeros(houses), np.zeros(houses, dtype=np.int32)
    _check(load().pcvg_simulate_radon(houses, counties, seed, _p(y), _p(x), _p(g, C.c_int32)))
    return Dataset(y, x.reshape(houses, 1), g)


def simulate_rat_growth(subjects=30, seed=1):
    """simulate_rat_growth (rat_growth.cpp:310-336): 5 weights per subject at t = 8..36."""
    n = 5 * subjects
    y, x, g = np.zeros(n), np.zeros(n), np.zeros(n, dtype=np.int32)
    _check(load().pcvg_simulate_rat(subjects, seed, _p(y), _p(x), _p(g, C.c_int32)))
    return Dataset(y, x.reshape(n, 1), g)


def simulate_seasonal_ar(months=432, ar_order=1, dummies=11, rho=0.6, seasonal_amp=1.0, sigma=1.0, seed=1):
    n = months - ar_order
    nc = ar_order + dummies
    y, x, t = np.zeros(n), np.zeros(n * nc), np.zeros(n, dtype=np.int64)
    _check(load().pcvg_simulate_seasonal(months, ar_order, dummies, rho, seasonal_amp, sigma, seed,
                                         _p(y), _p(x), _p(t, C.c_int64)))
    return Dataset(y, x.reshape(n, nc), None, t)


def simulate_linreg(n=100, covariates=5, seed=11):
    y, x, g = np.zeros(n), np.zeros(n * covariates), np.zeros(n, dtype=np.int32)
    _check(load().pcvg_simulate_linreg(n, covariates, seed, _p(y), _p(x), _p(g, C.c_int32)))
    return Dataset(y, x.reshape(n, covariates), g)


def simulate_logistic(n=10000, covariates=50, seed=1):
    y, x = np.zeros(n), np.zeros(n * covariates)
    _check(load().pcvg_simulate_logistic(n, covariates, seed, _p(y), _p(x)))
    return Dataset(y, x.reshape(n, covariates))


# ----------------------------------------------------------------- models (descriptors)
class Model:
    """A model descriptor: family + dataset + folds + options (the C-ABI replacement of a
    `pcv::Model*`, model.hpp:24-78)."""

    family = None

    def __init__(self, name, data, folds, **opts):
        self.name = name
        self.data = data
        self.folds = folds
        self.fold_arrays = folds.arrays()
        self.spec = abi.SpecArrays(self.family, **opts)

    @property
    def K(self):
        return self.folds.K

    def fold_count(self):
        return self.folds.K


class GroupedRegressionModel(Model):
    family = abi.FAMILY_GROUPED

    def __init__(self, name, data, folds, covariate_mask=None):
        super().__init__(name, data, folds, covariate_mask=covariate_mask)

    def dim(self):
        return self.data.n_groups + self.data.x.shape[1] + 3


class RadonStyleModel(Model):
    family = abi.FAMILY_RADON

    def __init__(self, name, data, folds, include_floor=True):
        super().__init__(name, data, folds, include_floor=int(include_floor))

    def dim(self):
        return self.data.n_groups + 4


class SeasonalARModel(Model):
    family = abi.FAMILY_SEASONAL_AR

    def __init__(self, name, data, folds, ar_order, seasonal_dummies, rho_transform=abi.RHO_HALF_OPEN):
        super().__init__(name, data, folds, ar_order=ar_order, dummies=seasonal_dummies,
                         rho_transform=rho_transform)
        self.p, self.q = ar_order, seasonal_dummies

    def dim(self):
        return self.p + self.q + 2


class RatGrowthModel(Model):
    """RatGrowthModel (rat_growth.hpp:20-63): per_subject_slope = M_A, else the shared-slope M_B."""
    family = abi.FAMILY_RAT_GROWTH

    def __init__(self, name, data, folds, per_subject_slope=True):
        super().__init__(name, data, folds, per_subject_slope=int(per_subject_slope))
        self.per_subject_slope = bool(per_subject_slope)

    def dim(self):
        J = self.data.n_groups
        return 2 * J + 5 if self.per_subject_slope else J + 4


class LogisticModel(Model):
    family = abi.FAMILY_LOGISTIC

    def dim(self):
        return self.data.x.shape[1] + 1


@dataclass
class KernelParams:
    step_size: float
    n_leapfrog: int
    inv_mass_diag: np.ndarray


@dataclass
class FullDataFit:
    """adapt.hpp:55-62: the tuned kernel and the draw bank (rows x dim)."""
    kparams: KernelParams
    draws: np.ndarray


@dataclass
class ModelInput:
    model: Model
    fit: FullDataFit
    model_id: int = 0


@dataclass
class AdaptConfig:
    """pcv::AdaptConfig (adapt.hpp:47-54)."""
    chains: int = 4
    warmup: int = 1000
    draws: int = 2000
    n_leapfrog: int = 32
    target_accept: float = 0.8
    init_step_size: float = 0.0


def RunConfig(**kw):
    """pcv::RunConfig defaults (engine.hpp:21-45) as a pcvg_run_config struct."""
    return abi.run_config(**kw)


# ----------------------------------------------------------------- device context
class Context:
    """One libpcvg context on one GPU (pcvg_create)."""

    def __init__(self, device=0):
        self.lib = load()
        self.h = C.c_void_p()
        _check(self.lib.pcvg_create(device, C.byref(self.h)))
        self.models = []
        self._keep = []

    def close(self):
        if self.h:
            self.lib.pcvg_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _chk(self, rc):
        _check(rc, self.h)

    def add_model(self, model, kparams, bank, model_id=0):
        kern = abi.KernelArrays(kparams.step_size, kparams.n_leapfrog, kparams.inv_mass_diag)
        bank = np.ascontiguousarray(bank, dtype=np.float64)
        slot = C.c_int32()
        self._chk(self.lib.pcvg_add_model(self.h, C.byref(model.data.struct),
                                          C.byref(model.fold_arrays.struct),
                                          C.byref(model.spec.struct), C.byref(kern.struct),
                                          _p(bank), bank.shape[0], model_id, C.byref(slot)))
        self.models.append(model)
        self._keep.append((kern, bank))
        return slot.value

    KERNEL_AUTO, KERNEL_GENERIC, KERNEL_TENSOR, KERNEL_TF32, KERNEL_SUFFSTAT, KERNEL_ROWS = 0, 1, 2, 3, 4, 5

    def debug_break_fold(self, slot, fold):
        """Tests only: every transition of fold `fold`'s chains diverges (BrokenFoldModel)."""
        self._chk(self.lib.pcvg_debug_break_fold(self.h, slot, fold))

    def set_kernel_policy(self, policy):
        self._chk(self.lib.pcvg_set_kernel_policy(self.h, policy))

    def adapt_full_data(self, model, cfg=None, seed=1, model_id=0, trace=False):
        """pcv::adapt_full_data (adapt.cpp:96-221) on the device: returns a FullDataFit with the
        tuned kernel and the (chains*draws) x dim bank, plus rhat / ess per parameter."""
        cfg = cfg or AdaptConfig()
        ac = abi.AdaptConfig(chains=cfg.chains, warmup=cfg.warmup, draws=cfg.draws,
                             n_leapfrog=cfg.n_leapfrog, target_accept=cfg.target_accept,
                             init_step_size=cfg.init_step_size)
        d = model.dim()
        im = np.zeros(d)
        bank = np.zeros((cfg.chains * cfg.draws, d))
        rh, es = np.zeros(d), np.zeros(d)
        st = np.zeros(cfg.warmup) if trace else None
        fit = abi.Fit(inv_mass_diag=_p(im), draws=_p(bank), rhat=_p(rh), ess=_p(es), step_trace=_p(st))
        self._chk(self.lib.pcvg_adapt_full_data(self.h, C.byref(model.data.struct),
                                                C.byref(model.fold_arrays.struct),
                                                C.byref(model.spec.struct), C.byref(ac), seed, model_id,
                                                C.byref(fit)))
        out = FullDataFit(KernelParams(fit.step_size, cfg.n_leapfrog, im), bank)
        out.rhat_per_param, out.ess_per_param = rh, es
        out.divergences, out.mean_accept, out.device_ms = fit.divergences, fit.mean_accept, fit.device_ms
        out.step_trace = st
        return out

    def dim(self, slot):
        d = C.c_int32()
        self._chk(self.lib.pcvg_model_dim(self.h, slot, C.byref(d)))
        return d.value

    def eval(self, slot, folds, thetas):
        """Model::log_joint + grad_log_joint at n points (device)."""
        folds = np.ascontiguousarray(np.atleast_1d(folds), dtype=np.int32)
        th = np.ascontiguousarray(np.atleast_2d(thetas), dtype=np.float64)
        n, d = th.shape
        lp, g = np.zeros(n), np.zeros((n, d))
        self._chk(self.lib.pcvg_eval(self.h, slot, n, _p(folds, C.c_int32), _p(th), _p(lp), _p(g)))
        return lp, g

    def eval_pred(self, slot, folds, thetas):
        folds = np.ascontiguousarray(np.atleast_1d(folds), dtype=np.int32)
        th = np.ascontiguousarray(np.atleast_2d(thetas), dtype=np.float64)
        out = np.zeros(th.shape[0])
        self._chk(self.lib.pcvg_eval_pred(self.h, slot, th.shape[0], _p(folds, C.c_int32), _p(th), _p(out)))
        return out

    def hmc_probe(self, slot, folds, thetas, momenta, us):
        folds = np.ascontiguousarray(np.atleast_1d(folds), dtype=np.int32)
        th = np.ascontiguousarray(np.atleast_2d(thetas), dtype=np.float64)
        mo = np.ascontiguousarray(np.atleast_2d(momenta), dtype=np.float64)
        u = np.ascontiguousarray(np.atleast_1d(us), dtype=np.float64)
        n = th.shape[0]
        out = np.zeros_like(th)
        h0, h1 = np.zeros(n), np.zeros(n)
        acc, div = np.zeros(n, dtype=np.int32), np.zeros(n, dtype=np.int32)
        self._chk(self.lib.pcvg_hmc_probe(self.h, slot, n, _p(folds, C.c_int32), _p(th), _p(mo), _p(u),
                                          _p(out), _p(h0), _p(h1), _p(acc, C.c_int32), _p(div, C.c_int32)))
        return out, h0, h1, acc, div

    def leapfrog(self, slot, folds, thetas, momenta):
        """leapfrog (hmc.cpp:22-51) end points (theta', p', ok) on the device."""
        folds = np.ascontiguousarray(np.atleast_1d(folds), dtype=np.int32)
        th = np.ascontiguousarray(np.atleast_2d(thetas), dtype=np.float64)
        mo = np.ascontiguousarray(np.atleast_2d(momenta), dtype=np.float64)
        n = th.shape[0]
        qo, po = np.zeros_like(th), np.zeros_like(th)
        ok = np.zeros(n, dtype=np.int32)
        self._chk(self.lib.pcvg_leapfrog(self.h, slot, n, _p(folds, C.c_int32), _p(th), _p(mo), _p(qo), _p(po),
                                         _p(ok, C.c_int32)))
        return qo, po, ok

    def hmc_chain(self, slot, fold, chain, seed, theta0, n_steps):
        th = np.ascontiguousarray(theta0, dtype=np.float64)
        traj = np.zeros((n_steps, th.shape[0]))
        div = np.zeros(n_steps, dtype=np.int32)
        self._chk(self.lib.pcvg_hmc_chain(self.h, slot, fold, chain, seed, _p(th), n_steps, _p(traj),
                                          _p(div, C.c_int32)))
        return traj, div

    def score_streams(self, streams, center=0.0, batch=10, blocks=5):
        """Feeds explicit per-chain log-score streams through the device accumulators and the fold
        reduction; returns dict(estimate, log_f_hat, mc, naive, ess, rhat, batches, fault)."""
        s = np.ascontiguousarray(np.atleast_2d(streams), dtype=np.float64)
        out = np.zeros(8)
        self._chk(self.lib.pcvg_score_streams(self.h, s.shape[0], s.shape[1], _p(s), center, batch,
                                              blocks, _p(out)))
        return dict(zip(["estimate", "log_f_hat", "mc", "naive", "ess", "rhat", "batches", "fault"], out))

    def run(self, cfg):
        K, L = self.models[0].K, cfg.chains
        nck = self.lib.pcvg_checkpoint_count(C.byref(cfg))
        rep, arrs = abi.new_report(len(self.models), K, L, nck, cfg.bench_draws)
        self._chk(self.lib.pcvg_run(self.h, C.byref(cfg), C.byref(rep)))
        return abi.report_dict(rep, arrs, len(self.models))

    def run_streams(self, scores, centers, cfg):
        """pcvg_run_streams: run_pcv's checkpoints, per-fold statistics, shuffle benchmark and early-stop
        rule on explicit log_pred streams scores[K][L][iters] (fold centres centers[K]) instead of
        sampled ones; needs a context without models."""
        s = np.ascontiguousarray(scores, dtype=np.float64)
        K, L, n = s.shape
        if L != cfg.chains or n != cfg.iters:
            raise InvalidInput("scores must be [K][chains][iters]")
        c = np.ascontiguousarray(centers, dtype=np.float64)
        nck = self.lib.pcvg_checkpoint_count(C.byref(cfg))
        rep, arrs = abi.new_report(1, K, L, nck, cfg.bench_draws)
        self._chk(self.lib.pcvg_run_streams(self.h, K, _p(s), _p(c), C.byref(cfg), C.byref(rep)))
        return abi.report_dict(rep, arrs, 1)

    # stepwise API (sharded runs)
    def begin(self, cfg):
        self._cfg = cfg
        self._chk(self.lib.pcvg_begin(self.h, C.byref(cfg)))

    def advance(self, n_iters):
        self._chk(self.lib.pcvg_advance(self.h, n_iters))

    def last_advance_ms(self):
        ms, n = C.c_double(), C.c_int64()
        self._chk(self.lib.pcvg_timing(self.h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def fold_stats(self, nfold):
        nm = len(self.models)
        ft, cols = abi.new_fold_table(nm * nfold)
        div = np.zeros(nm * nfold * self._cfg.chains, dtype=np.int64)
        dropped, done = C.c_int64(), C.c_int64()
        self._chk(self.lib.pcvg_fold_stats(self.h, C.byref(ft), _p(div, C.c_int64), C.byref(dropped),
                                           C.byref(done)))
        return cols, div, dropped.value, done.value

    def benchmark(self, failed=None, nonfailed_before=0, nonfailed_total=None, blocks_used=None):
        """pcvg_benchmark: the shard's shuffle-benchmark replicate maxima on device."""
        R = self._cfg.bench_draws
        nfold = (self._cfg.fold_end - self._cfg.fold_begin) or self.models[0].K
        if nonfailed_total is None:
            nonfailed_total = nfold if failed is None else int(np.sum(np.asarray(failed) == 0))
        fl = None if failed is None else np.ascontiguousarray(failed, dtype=np.int32)
        mx, nh = np.zeros(R), np.zeros(R, dtype=np.int32)
        self._chk(self.lib.pcvg_benchmark(self.h, _p(fl, C.c_int32), nonfailed_before, nonfailed_total,
                                          blocks_used or self._cfg.blocks, _p(mx), _p(nh, C.c_int32)))
        return mx, nh

    def block_sums(self, nfold, D):
        nm = len(self.models)
        n = nm * nfold * self._cfg.chains * D
        a, b = np.zeros(n), np.zeros(n)
        self._chk(self.lib.pcvg_block_sums(self.h, _p(a), _p(b)))
        return a, b


class MultiContext:
    """run_pcv across several devices in one process (pcvg_multi_*): folds sharded in contiguous
    ranges, one host thread per device, per-fold tables merged in fold order. Device ids may repeat
    (several shards on one GPU)."""

    def __init__(self, devices):
        self.lib = load()
        ids = np.ascontiguousarray(devices, dtype=np.int32)
        self.h = C.c_void_p()
        rc = self.lib.pcvg_multi_create(len(ids), _p(ids, C.c_int32), C.byref(self.h))
        if rc != 0:
            _check(rc)
        self.models = []
        self._keep = []

    def close(self):
        if self.h:
            self.lib.pcvg_multi_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _chk(self, rc):
        if rc != 0:
            raise _EXC.get(rc, PcvError)(self.lib.pcvg_multi_last_error(self.h).decode())

    def set_kernel_policy(self, policy):
        self._chk(self.lib.pcvg_multi_set_kernel_policy(self.h, policy))

    def add_model(self, model, kparams, bank, model_id=0):
        kern = abi.KernelArrays(kparams.step_size, kparams.n_leapfrog, kparams.inv_mass_diag)
        bank = np.ascontiguousarray(bank, dtype=np.float64)
        slot = C.c_int32()
        self._chk(self.lib.pcvg_multi_add_model(self.h, C.byref(model.data.struct), C.byref(model.fold_arrays.struct),
                                                C.byref(model.spec.struct), C.byref(kern.struct), _p(bank),
                                                bank.shape[0], model_id, C.byref(slot)))
        self.models.append(model)
        self._keep.append((kern, bank))
        return slot.value

    def run(self, cfg):
        K, L = self.models[0].K, cfg.chains
        nck = self.lib.pcvg_checkpoint_count(C.byref(cfg))
        rep, arrs = abi.new_report(len(self.models), K, L, nck, cfg.bench_draws)
        self._chk(self.lib.pcvg_multi_run(self.h, C.byref(cfg), C.byref(rep)))
        return abi.report_dict(rep, arrs, len(self.models))


def merge(n_models, K, cfg, iter_count, final, cols, y_x=None, y_x2=None):
    """pcvg_merge: Step-4 statistics from full fold-order tables (all shards)."""
    lib = load()
    ft = abi.FoldTable(**{name: abi.ptr(np.ascontiguousarray(cols[name]), abi._CT[dt])
                          for name, dt in abi.FOLD_COLUMNS})
    rep, arrs = abi.new_report(n_models, K, cfg.chains, 1, cfg.bench_draws)
    _check(lib.pcvg_merge(n_models, K, C.byref(cfg), iter_count, int(final), C.byref(ft),
                          None if y_x is None else _p(y_x), None if y_x2 is None else _p(y_x2),
                          C.byref(rep)))
    return abi.report_dict(rep, arrs, n_models)


def benchmark_host(n_models, nfold, L, D_stride, blocks_used, iter_count, seed, bench_draws, y_x, y_x2,
                   failed=None, nonfailed_before=0, nonfailed_total=None, block_groups=None):
    """pcvg_benchmark_host: positional shuffle benchmark of one shard from host sub-block sums (the
    first blocks_used sub-blocks regrouped into block_groups blocks; default: one each)."""
    if nonfailed_total is None:
        nonfailed_total = nfold if failed is None else int(np.sum(np.asarray(failed) == 0))
    fl = None if failed is None else np.ascontiguousarray(failed, dtype=np.int32)
    mx, nh = np.zeros(bench_draws), np.zeros(bench_draws, dtype=np.int32)
    _check(load().pcvg_benchmark_host(n_models, nfold, L, D_stride, blocks_used, block_groups or blocks_used,
                                      iter_count, seed, bench_draws,
                                      _p(np.ascontiguousarray(y_x)), _p(np.ascontiguousarray(y_x2)),
                                      _p(fl, C.c_int32), nonfailed_before, nonfailed_total, _p(mx),
                                      _p(nh, C.c_int32)))
    return mx, nh


def merge_bench(n_models, K, cfg, iter_count, final, cols, bench_max):
    """pcvg_merge_bench: Step-4 statistics with precomputed benchmark replicate maxima."""
    lib = load()
    ft = abi.FoldTable(**{name: abi.ptr(np.ascontiguousarray(cols[name]), abi._CT[dt])
                          for name, dt in abi.FOLD_COLUMNS})
    rep, arrs = abi.new_report(n_models, K, cfg.chains, 1, cfg.bench_draws)
    bm = np.ascontiguousarray(bench_max, dtype=np.float64)
    _check(lib.pcvg_merge_bench(n_models, K, C.byref(cfg), iter_count, int(final), C.byref(ft), _p(bm),
                                C.byref(rep)))
    return abi.report_dict(rep, arrs, n_models)


def fold_gram(y, x, key, lo, hi):
    """pcvg_fold_gram (host): packed training Gram of u = (y, x) for every fold and the sentinel."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    n = y.size
    x = np.asarray(x, dtype=np.float64).reshape(n, -1)
    nc = x.shape[1]
    xc = np.ascontiguousarray(x.T)
    key = np.ascontiguousarray(key, dtype=np.int32)
    lo = np.ascontiguousarray(lo, dtype=np.int32)
    hi = np.ascontiguousarray(hi, dtype=np.int32)
    K = lo.size
    dp = (nc + 1) * (nc + 2) // 2
    out = np.zeros((K + 1) * dp)
    _check(load().pcvg_fold_gram(n, nc, _p(y), _p(xc), _p(key, C.c_int32), K, _p(lo, C.c_int32), _p(hi, C.c_int32),
                                 _p(out)))
    return out.reshape(K + 1, dp)


def initial_draw(model, seed, stream):
    """Model::initial_draw (model.hpp:44) on CounterRng(seed, stream) (host, bit-exact)."""
    out = np.zeros(model.dim())
    _check(load().pcvg_initial_draw(C.byref(model.data.struct), C.byref(model.fold_arrays.struct),
                                    C.byref(model.spec.struct), seed, stream, _p(out)))
    return out


def adapt_full_data(model, cfg=None, seed=1, model_id=0, device=0):
    """pcv::adapt_full_data (adapt.hpp:64-69) on one GPU."""
    with Context(device) as ctx:
        return ctx.adapt_full_data(model, cfg, seed, model_id)


def run_pcv(inputs, cfg, device=0):
    """pcv::run_pcv (engine.cpp:257-483) on one GPU."""
    with Context(device) as ctx:
        for mi in inputs:
            ctx.add_model(mi.model, mi.fit.kparams, mi.fit.draws, mi.model_id)
        return ctx.run(cfg)

"""Loaders for the CPU oracle (tests only).

* liboracle.so  - oracle/pcv_oracle.c, the C restatement (always buildable; travels to the box)
* libpcvref.so  - the reference library compiled in place from /root/reference (oracle/_ref/)
"""
import ctypes as C
import os

import numpy as np

from paper_2310_07002_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libpcvref.so")

f64, i32, i64, u64 = C.c_double, C.c_int32, C.c_int64, C.c_uint64
pf64, pi32, pi64, pu64 = abi.P_f64, abi.P_i32, abi.P_i64, abi.P_u64
vp = C.c_void_p


def _sig(lib, name, res, args):
    fn = getattr(lib, name)
    fn.restype = res
    fn.argtypes = args
    return fn


_oracle = None
_ref = None


def oracle():
    global _oracle
    if _oracle is None:
        lib = C.CDLL(ORACLE_SO)
        P = C.POINTER
        _sig(lib, "pcvo_stream_key", u64, [u64, u64, u64, u64])
        _sig(lib, "pcvo_rng_sequence", C.c_int, [u64, u64, i32, u64, C.c_char_p, pu64, i64, pf64])
        _sig(lib, "pcvo_make_kfold", C.c_int, [i64, i32, u64, pi32])
        _sig(lib, "pcvo_make_time_blocks", C.c_int, [P(abi.Dataset), i32, pi32])
        _sig(lib, "pcvo_make_hv_block", C.c_int, [P(abi.Dataset), i32, i64, pi64])
        _sig(lib, "pcvo_make_hv_racine", C.c_int, [P(abi.Dataset), i64, i64, pi64])
        _sig(lib, "pcvo_model_create", vp, [P(abi.Dataset), P(abi.Folds), P(abi.ModelSpec)])
        _sig(lib, "pcvo_model_destroy", None, [vp])
        _sig(lib, "pcvo_model_break_fold", None, [vp, i32])
        _sig(lib, "pcvo_model_dim", i32, [vp])
        _sig(lib, "pcvo_test_size", i64, [vp, i32])
        _sig(lib, "pcvo_log_joint", f64, [vp, pf64, i32])
        _sig(lib, "pcvo_grad", None, [vp, pf64, i32, pf64])
        _sig(lib, "pcvo_log_pred", f64, [vp, pf64, i32])
        _sig(lib, "pcvo_leapfrog", i32, [vp, i32, f64, i32, pf64, pf64, pf64])
        _sig(lib, "pcvo_hmc_probe", None, [vp, i32, f64, i32, pf64, pf64, pf64, f64, pf64, pf64,
                                            pf64, pi32, pi32])
        _sig(lib, "pcvo_hmc_chain", C.c_int, [vp, i32, f64, i32, pf64, u64, u64, pf64, i64, pf64, pi32])
        _sig(lib, "pcvo_run_pcv", C.c_int, [i32, P(vp), pi32, P(abi.Kernel), P(pf64), pi64,
                                             P(abi.RunConfig), i32, P(abi.Report), vp, i32])
        _sig(lib, "pcvo_rhat_from_sums", C.c_int, [pf64, pf64, i32, i64, pf64, pf64, pf64])
        _sig(lib, "pcvo_selection_probability", f64, [f64, pf64, i64, pf64])
        _sig(lib, "pcvo_benchmark_quantile", f64, [pf64, i64, f64])
        _sig(lib, "pcvo_time_tasks", C.c_int, [vp, i32, pi32, i32, i64, i64, u64, i32, P(abi.Kernel), pf64,
                                                i64, i32, pf64, pf64, pf64])
        _sig(lib, "pcvo_score_streams", C.c_int, [i32, i64, pf64, f64, i32, i32, pf64])
        _sig(lib, "pcvo_supports_pred", C.c_int, [vp])
        _sig(lib, "pcvo_pred_derivs", None, [vp, pf64, i32, pf64, pf64])
        _sig(lib, "pcvo_pred_sample_stream", C.c_int, [vp, pf64, i32, u64, u64, i32, pf64])
        _sig(lib, "pcvo_last_error", C.c_char_p, [])
        _oracle = lib
    return _oracle


def have_ref():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        P = C.POINTER
        _sig(lib, "pcvref_last_error", C.c_char_p, [])
        _sig(lib, "pcvref_stream_key", u64, [u64, u64, u64, u64])
        _sig(lib, "pcvref_rng_sequence", C.c_int, [u64, u64, i32, u64, C.c_char_p, pu64, i64, pf64])
        _sig(lib, "pcvref_make_kfold", C.c_int, [i64, i32, u64, pi32])
        _sig(lib, "pcvref_make_time_blocks", C.c_int, [P(abi.Dataset), i32, pi32])
        _sig(lib, "pcvref_make_logo", C.c_int, [P(abi.Dataset), pi32, pi32])
        _sig(lib, "pcvref_simulate_grouped", C.c_int, [i32, i32, i32, f64, u64, pf64, pf64, pi32])
        _sig(lib, "pcvref_simulate_radon", C.c_int, [i32, i32, u64, pf64, pf64, pi32])
        _sig(lib, "pcvref_simulate_seasonal", C.c_int, [i64, i32, i32, f64, f64, f64, u64, pf64, pf64, pi64])
        _sig(lib, "pcvref_model_create", vp, [P(abi.Dataset), P(abi.Folds), P(abi.ModelSpec), C.c_char_p])
        _sig(lib, "pcvref_model_destroy", None, [vp])
        _sig(lib, "pcvref_model_dim", i32, [vp])
        _sig(lib, "pcvref_test_size", i64, [vp, i32])
        _sig(lib, "pcvref_log_joint", f64, [vp, pf64, i32])
        _sig(lib, "pcvref_grad", None, [vp, pf64, i32, pf64])
        _sig(lib, "pcvref_log_pred", f64, [vp, pf64, i32])
        _sig(lib, "pcvref_log_lik_test", f64, [vp, pf64, i32])
        _sig(lib, "pcvref_initial_draw", None, [vp, u64, u64, pf64])
        _sig(lib, "pcvref_pred_derivs", C.c_int, [vp, pf64, i32, pf64, pf64])
        _sig(lib, "pcvref_adapt_trace", C.c_int, [vp, i32, i64, i32, f64, u64, i32, pf64, pf64, pf64,
                                                   pf64, pf64])
        _sig(lib, "pcvref_pred_sample", C.c_int, [vp, pf64, i32, u64, u64, i32, pf64])
        _sig(lib, "pcvref_leapfrog", i32, [vp, i32, f64, i32, pf64, pf64, pf64])
        _sig(lib, "pcvref_hmc_chain", C.c_int, [vp, i32, f64, i32, pf64, u64, u64, pf64, i64, pf64,
                                                 pi32, pi32, pf64])
        _sig(lib, "pcvref_adapt", C.c_int, [vp, i32, i64, i64, i32, f64, f64, u64, i32, pf64, pf64,
                                             pf64, pf64, pi64])
        _sig(lib, "pcvref_time_tasks", C.c_int, [vp, i32, pi32, i32, i64, i64, u64, i32, P(abi.Kernel), pf64,
                                                  i64, i32, pf64, pf64, pf64])
        _sig(lib, "pcvref_run_pcv", C.c_int, [i32, P(vp), pi32, P(abi.Kernel), P(pf64), pi64,
                                               P(abi.RunConfig), i32, P(abi.Report)])
        _ref = lib
    return _ref


def _p(a, ct=C.c_double):
    return abi.ptr(a, ct)


class OModel:
    """An oracle (C restatement) model built from the same descriptor as the product."""

    def __init__(self, data, folds, spec, lib=None):
        self.lib = lib or oracle()
        self.data, self.folds, self.spec = data, folds, spec
        self.h = self.lib.pcvo_model_create(C.byref(data.struct), C.byref(folds.struct), C.byref(spec.struct))
        if not self.h:
            raise ValueError(self.lib.pcvo_last_error().decode())
        self.dim = self.lib.pcvo_model_dim(self.h)
        self.K = folds.K

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.pcvo_model_destroy(self.h)

    def break_fold(self, fold):
        """BrokenFoldModel (test_engine.cpp:57-90): NaN gradient on `fold` (-1 clears)."""
        self.lib.pcvo_model_break_fold(self.h, fold)

    def log_joint(self, th, fold):
        th = np.ascontiguousarray(th, dtype=np.float64)
        return self.lib.pcvo_log_joint(self.h, _p(th), fold)

    def grad(self, th, fold):
        th = np.ascontiguousarray(th, dtype=np.float64)
        g = np.zeros(self.dim)
        self.lib.pcvo_grad(self.h, _p(th), fold, _p(g))
        return g

    def log_pred(self, th, fold):
        th = np.ascontiguousarray(th, dtype=np.float64)
        return self.lib.pcvo_log_pred(self.h, _p(th), fold)

    def test_size(self, fold):
        return self.lib.pcvo_test_size(self.h, fold)

    def pred_derivs(self, th, fold):
        th = np.ascontiguousarray(th, dtype=np.float64)
        n = self.test_size(fold)
        d1, d2 = np.zeros(max(n, 1)), np.zeros(max(n, 1))
        self.lib.pcvo_pred_derivs(self.h, _p(th), fold, _p(d1), _p(d2))
        return d1[:n], d2[:n]

    def pred_sample(self, th, fold, seed, stream, times=1):
        th = np.ascontiguousarray(th, dtype=np.float64)
        n = self.test_size(fold)
        out = np.zeros(max(n * times, 1))
        rc = self.lib.pcvo_pred_sample_stream(self.h, _p(th), fold, seed, stream, times, _p(out))
        assert rc == 0
        return out[:n * times].reshape(times, n)

    def leapfrog(self, fold, step, n_lf, inv_mass, q, p):
        q = np.array(q, dtype=np.float64)
        p = np.array(p, dtype=np.float64)
        im = np.ascontiguousarray(inv_mass, dtype=np.float64)
        ok = self.lib.pcvo_leapfrog(self.h, fold, step, n_lf, _p(im), _p(q), _p(p))
        return ok, q, p

    def hmc_probe(self, fold, step, n_lf, inv_mass, theta, momentum, u):
        im = np.ascontiguousarray(inv_mass, dtype=np.float64)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        mo = np.ascontiguousarray(momentum, dtype=np.float64)
        out = np.zeros(self.dim)
        h0, h1 = f64(), f64()
        acc, div = i32(), i32()
        self.lib.pcvo_hmc_probe(self.h, fold, step, n_lf, _p(im), _p(th), _p(mo), u, _p(out),
                                C.byref(h0), C.byref(h1), C.byref(acc), C.byref(div))
        return out, h0.value, h1.value, acc.value, div.value

    def hmc_chain(self, fold, step, n_lf, inv_mass, seed, stream, theta0, n_steps):
        im = np.ascontiguousarray(inv_mass, dtype=np.float64)
        th = np.ascontiguousarray(theta0, dtype=np.float64)
        traj = np.zeros((n_steps, self.dim))
        div = np.zeros(n_steps, dtype=np.int32)
        self.lib.pcvo_hmc_chain(self.h, fold, step, n_lf, _p(im), seed, stream, _p(th), n_steps,
                                _p(traj), _p(div, C.c_int32))
        return traj, div


class RModel:
    """The reference's own Model (or an oracle plugin on the reference API)."""

    def __init__(self, data, folds, spec, name=b"M"):
        self.lib = ref()
        self.h = self.lib.pcvref_model_create(C.byref(data.struct), C.byref(folds.struct),
                                              C.byref(spec.struct), name)
        if not self.h:
            raise ValueError(self.lib.pcvref_last_error().decode())
        self.dim = self.lib.pcvref_model_dim(self.h)
        self.K = folds.K

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.pcvref_model_destroy(self.h)

    def log_joint(self, th, fold):
        th = np.ascontiguousarray(th, dtype=np.float64)
        return self.lib.pcvref_log_joint(self.h, _p(th), fold)

    def grad(self, th, fold):
        th = np.ascontiguousarray(th, dtype=np.float64)
        g = np.zeros(self.dim)
        self.lib.pcvref_grad(self.h, _p(th), fold, _p(g))
        return g

    def log_pred(self, th, fold):
        th = np.ascontiguousarray(th, dtype=np.float64)
        return self.lib.pcvref_log_pred(self.h, _p(th), fold)

    def log_lik_test(self, th, fold):
        th = np.ascontiguousarray(th, dtype=np.float64)
        return self.lib.pcvref_log_lik_test(self.h, _p(th), fold)

    def test_size(self, fold):
        return self.lib.pcvref_test_size(self.h, fold)

    def pred_derivs(self, th, fold):
        th = np.ascontiguousarray(th, dtype=np.float64)
        n = self.test_size(fold)
        d1, d2 = np.zeros(max(n, 1)), np.zeros(max(n, 1))
        assert self.lib.pcvref_pred_derivs(self.h, _p(th), fold, _p(d1), _p(d2)) == 0
        return d1[:n], d2[:n]

    def pred_sample(self, th, fold, seed, stream, times=1):
        th = np.ascontiguousarray(th, dtype=np.float64)
        n = self.test_size(fold)
        out = np.zeros(max(n * times, 1))
        assert self.lib.pcvref_pred_sample(self.h, _p(th), fold, seed, stream, times, _p(out)) == 0
        return out[:n * times].reshape(times, n)

    def initial_draw(self, seed, stream):
        out = np.zeros(self.dim)
        self.lib.pcvref_initial_draw(self.h, seed, stream, _p(out))
        return out

    def leapfrog(self, fold, step, n_lf, inv_mass, q, p):
        q = np.array(q, dtype=np.float64)
        p = np.array(p, dtype=np.float64)
        im = np.ascontiguousarray(inv_mass, dtype=np.float64)
        ok = self.lib.pcvref_leapfrog(self.h, fold, step, n_lf, _p(im), _p(q), _p(p))
        return ok, q, p

    def hmc_chain(self, fold, step, n_lf, inv_mass, seed, stream, theta0, n_steps):
        im = np.ascontiguousarray(inv_mass, dtype=np.float64)
        th = np.ascontiguousarray(theta0, dtype=np.float64)
        traj = np.zeros((n_steps, self.dim))
        div = np.zeros(n_steps, dtype=np.int32)
        acc = np.zeros(n_steps, dtype=np.int32)
        dh = np.zeros(n_steps)
        rc = self.lib.pcvref_hmc_chain(self.h, fold, step, n_lf, _p(im), seed, stream, _p(th),
                                       n_steps, _p(traj), _p(div, C.c_int32), _p(acc, C.c_int32), _p(dh))
        assert rc == 0, self.lib.pcvref_last_error()
        return traj, div

    def adapt_trace(self, chains=4, warmup=30, n_lf=32, target=0.8, seed=1, model_id=0):
        init = f64()
        st, ap = np.zeros(warmup), np.zeros(warmup)
        im = np.zeros(self.dim)
        pos = np.zeros((chains, self.dim))
        rc = self.lib.pcvref_adapt_trace(self.h, chains, warmup, n_lf, target, seed, model_id, C.byref(init),
                                         _p(st), _p(ap), _p(im), _p(pos))
        assert rc == 0, self.lib.pcvref_last_error()
        return dict(init_step=init.value, step_trace=st, ap_trace=ap, inv_mass=im, start=pos)

    def adapt(self, chains=4, warmup=1000, draws=2000, n_lf=32, target=0.8, init_step=0.0,
              seed=1, model_id=0):
        step = f64()
        inv_mass = np.zeros(self.dim)
        bank = np.zeros((chains * draws, self.dim))
        acc = f64()
        div = i64()
        rc = self.lib.pcvref_adapt(self.h, chains, warmup, draws, n_lf, target, init_step, seed,
                                   model_id, C.byref(step), _p(inv_mass), _p(bank), C.byref(acc),
                                   C.byref(div))
        if rc != 0:
            raise RuntimeError(self.lib.pcvref_last_error().decode())
        return {"step_size": step.value, "n_leapfrog": n_lf, "inv_mass_diag": inv_mass,
                "bank": bank, "mean_accept": acc.value, "divergences": div.value}


def _run(lib_fn, handles, model_ids, kernels, banks, cfg, threads, extra=()):
    n_models = len(handles)
    K = None
    arr_h = (vp * n_models)(*handles)
    ks = (abi.Kernel * n_models)(*[k.struct for k in kernels])
    banks = [np.ascontiguousarray(b, dtype=np.float64) for b in banks]
    bptr = (pf64 * n_models)(*[_p(b) for b in banks])
    rows = np.array([b.shape[0] for b in banks], dtype=np.int64)
    ids = np.array(model_ids, dtype=np.int32)
    return arr_h, ks, bptr, rows, ids, banks


def run_pcv_oracle(models, model_ids, kernels, banks, cfg, threads=0):
    """pcvo_run_pcv: the C restatement of run_pcv. models: list of OModel."""
    lib = models[0].lib
    K, L = models[0].K, cfg.chains
    rep, arrs = abi.new_report(len(models), K, L, abi.checkpoint_count(cfg.iters, cfg.checkpoint_every),
                               cfg.bench_draws)
    arr_h, ks, bptr, rows, ids, keep = _run(None, [m.h for m in models], model_ids, kernels, banks, cfg, threads)
    rc = lib.pcvo_run_pcv(len(models), arr_h, _p(ids, C.c_int32), ks, bptr, _p(rows, C.c_int64),
                          C.byref(cfg), threads, C.byref(rep), None, 0)
    if rc != 0:
        raise RuntimeError(lib.pcvo_last_error().decode())
    return abi.report_dict(rep, arrs, len(models))


def run_pcv_ref(models, model_ids, kernels, banks, cfg, threads=0):
    """pcvref_run_pcv: the reference engine itself."""
    lib = ref()
    K, L = models[0].K, cfg.chains
    rep, arrs = abi.new_report(len(models), K, L, abi.checkpoint_count(cfg.iters, cfg.checkpoint_every),
                               cfg.bench_draws)
    arrs["naive_contribution"][:] = np.nan
    arr_h, ks, bptr, rows, ids, keep = _run(None, [m.h for m in models], model_ids, kernels, banks, cfg, threads)
    rc = lib.pcvref_run_pcv(len(models), arr_h, _p(ids, C.c_int32), ks, bptr, _p(rows, C.c_int64),
                            C.byref(cfg), threads, C.byref(rep))
    if rc != 0:
        raise RuntimeError(lib.pcvref_last_error().decode())
    return abi.report_dict(rep, arrs, len(models))

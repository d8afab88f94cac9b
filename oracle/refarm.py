"""TEST / BASELINE INFRASTRUCTURE ONLY: the CPU arms of bench.py.

Times the reference's own Step 2-3 task loop (engine.cpp:296-381 via oracle/ref_shim.cpp
`pcvref_time_tasks`: warm start, warmup_discard, then hmc_step + log_pred + ScoreAccum::observe,
on the reference thread pool) on a bounded fold sample of the cfg2 workload. Everything comes from
oracle/_ref/libpcvref.so (the reference compiled in place) - the dataset is simulated there
(`pcvref_simulate_logistic`, same draws as the product simulator; pinned by
tests/test_oracle_pinning.py), the kernel and draw bank are read from the committed fixture with
numpy. Nothing here imports or loads the product package (paper_2310_07002_b200 / libpcvg.so).
When the reference build is absent the C restatement (oracle/_build/liboracle.so) is timed instead.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF_SO = os.path.join(HERE, "_ref", "libpcvref.so")
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
FIXTURE = os.path.join(ROOT, "tests", "golden", "cfg2_logistic_bench.npz")

PF64, PI32, PI64 = C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_int64)
FAMILY_LOGISTIC = 3


# The four plain structs of include/pcvg.h the CPU arms need (pcvg_dataset, pcvg_folds,
# pcvg_model_spec, pcvg_kernel); the oracle and the reference shim compile against that header.
class Dataset(C.Structure):
    _fields_ = [("n_obs", C.c_int64), ("n_cov", C.c_int32), ("y", PF64), ("x", PF64),
                ("group_id", PI32), ("time_index", PI64)]


class Folds(C.Structure):
    _fields_ = [("K", C.c_int32), ("test_index", PI32), ("intervals", PI64)]


class ModelSpec(C.Structure):
    _fields_ = [("family", C.c_int32), ("covariate_mask", PI32), ("include_floor", C.c_int32),
                ("ar_order", C.c_int32), ("dummies", C.c_int32), ("rho_transform", C.c_int32),
                ("per_subject_slope", C.c_int32)]


class Kernel(C.Structure):
    _fields_ = [("step_size", C.c_double), ("n_leapfrog", C.c_int32), ("inv_mass_diag", PF64)]


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def have_ref():
    return os.path.exists(REF_SO)


def load_fixture():
    """(n_obs, covariates, seed, step_size, inv_mass_diag, bank) of the cfg2 bench fixture."""
    z = np.load(FIXTURE)
    n, p, seed = (int(v) for v in (z["sim_logistic"] if "sim_logistic" in z else z["sim_args"]))
    return n, p, seed, float(z["step0"]), np.ascontiguousarray(z["inv_mass0"]), np.ascontiguousarray(z["bank0"])


class Workload:
    """The cfg2 model (logistic, LOO) built inside the CPU library."""

    def __init__(self, prefer_ref=True):
        self.kind = "reference" if (prefer_ref and have_ref()) else "port"
        self.lib = C.CDLL(REF_SO if self.kind == "reference" else ORACLE_SO)
        pre = "pcvref_" if self.kind == "reference" else "pcvo_"
        self.f_create = getattr(self.lib, pre + "model_create")
        self.f_create.restype = C.c_void_p
        self.f_destroy = getattr(self.lib, pre + "model_destroy")
        self.f_destroy.argtypes = [C.c_void_p]
        self.f_time = getattr(self.lib, pre + "time_tasks")
        self.f_time.restype = C.c_int
        self.f_time.argtypes = [C.c_void_p, C.c_int32, PI32, C.c_int32, C.c_int64, C.c_int64, C.c_uint64,
                                C.c_int32, C.POINTER(Kernel), PF64, C.c_int64, C.c_int32, PF64, PF64, PF64]
        n, p, seed, step, inv_mass, bank = load_fixture()
        self.n, self.p = n, p
        self.y = np.zeros(n)
        self.x = np.zeros(n * p)
        if self.kind == "reference":
            sim = self.lib.pcvref_simulate_logistic
            sim.restype = C.c_int
            sim.argtypes = [C.c_int64, C.c_int32, C.c_uint64, PF64, PF64]
            rc = sim(n, p, seed, _ptr(self.y, C.c_double), _ptr(self.x, C.c_double))
        else:
            sim = self.lib.pcvo_simulate_logistic
            sim.restype = C.c_int
            sim.argtypes = [C.c_int64, C.c_int32, C.c_uint64, PF64, PF64]
            rc = sim(n, p, seed, _ptr(self.y, C.c_double), _ptr(self.x, C.c_double))
        assert rc == 0, "logistic simulator failed"
        self.test_index = np.arange(n, dtype=np.int32)  # LOO (folds.cpp:43-52)
        self.ds = Dataset(n, p, _ptr(self.y, C.c_double), _ptr(self.x, C.c_double), None, None)
        self.fs = Folds(n, _ptr(self.test_index, C.c_int32), None)
        self.spec = ModelSpec(FAMILY_LOGISTIC, None, 1, 1, 0, 0, 0)
        args = [C.byref(self.ds), C.byref(self.fs), C.byref(self.spec)]
        if self.kind == "reference":
            args.append(b"M_A")
        self.f_create.argtypes = [C.POINTER(Dataset), C.POINTER(Folds), C.POINTER(ModelSpec)] + (
            [C.c_char_p] if self.kind == "reference" else [])
        self.h = self.f_create(*args)
        assert self.h, "model creation failed"
        self.inv_mass = inv_mass
        self.bank = bank
        self.kern = Kernel(step, 32, _ptr(self.inv_mass, C.c_double))

    def time_tasks(self, folds, L, warmup, steps, threads, seed=1):
        folds = np.ascontiguousarray(folds, dtype=np.int32)
        s_s, w_s, cs = C.c_double(), C.c_double(), C.c_double()
        rc = self.f_time(self.h, len(folds), _ptr(folds, C.c_int32), L, warmup, steps, seed, 0,
                         C.byref(self.kern), _ptr(self.bank, C.c_double), self.bank.shape[0], threads,
                         C.byref(s_s), C.byref(w_s), C.byref(cs))
        assert rc == 0, "cpu task loop failed"
        return s_s.value, w_s.value, cs.value

    def close(self):
        if self.h:
            self.f_destroy(self.h)
            self.h = None


def cpu_sample(folds_total, n_sample_folds, L, steps, warmup, threads, prefer_ref=True):
    """(chain-steps/s, kind, sample description) of the CPU task loop on a seeded fold sample."""
    w = Workload(prefer_ref)
    rng = np.random.default_rng(0)
    folds = np.sort(rng.choice(folds_total, n_sample_folds, replace=False)).astype(np.int32)
    secs, _, _ = w.time_tasks(folds, L, warmup, steps, threads)
    w.close()
    chain_steps = len(folds) * L * steps
    sample = (f"{len(folds)} of {folds_total} LOO folds x {L} chains x {steps} sampling steps "
              f"(after {warmup} warm-up steps) = {chain_steps} chain-steps, {threads} threads, {secs:.2f} s")
    return chain_steps / secs, w.kind, sample

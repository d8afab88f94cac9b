"""The fold-sharded multi-process driver (dist.run_pcv_sharded) on real device runs: two ranks, each a
process with its own pcvg context on cuda:0, exchanging their per-fold tables and benchmark maxima
over gloo (host collectives: no kernel of one rank waits on the other). Against the unsharded
pcvg_run on the same inputs (the reference's thread-count invariance, test_engine.cpp:106-148, as
GPU-count invariance):

* Gaussian families on the sufficient-statistics kernel (one chain per thread, geometry-independent
  arithmetic): every per-fold column, the divergences, the benchmark replicates and the headline
  statistics are bit-identical, with and without the early-stop rule;
* logistic (tensor-core GLM kernel, whose row-split cluster size follows the shard's tile count):
  per-fold estimates equal to rounding at a short horizon, Delta-hat within Monte Carlo error.
"""
import os
import pickle
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import os, pickle, sys
sys.path[:0] = ["tests", "tests/golden", "."]
import torch.distributed as tdist
from parity_util import Case
from paper_2310_07002_b200 import abi, dist, pcv
name, cfgkw, out, backend = sys.argv[1], eval(sys.argv[2]), sys.argv[3], sys.argv[4]
if backend == "nccl":
    import torch
    torch.cuda.set_device(0)
    tdist.init_process_group("nccl", device_id=torch.device("cuda", 0))
else:
    tdist.init_process_group("gloo")
case = Case(name)
inputs = [pcv.ModelInput(m, pcv.FullDataFit(kp, bank), i)
          for i, (m, kp, bank) in enumerate(zip(case.models, case.kparams, case.banks))]
rep = dist.run_pcv_sharded(inputs, abi.run_config(**cfgkw), device=0)
if tdist.get_rank() == 0:
    with open(out, "wb") as f:
        pickle.dump(rep, f)
tdist.barrier()
tdist.destroy_process_group()
'''


def run_sharded(name, cfgkw, world=2, backend="gloo"):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as tmp:
        out = os.path.join(tmp, "rep.pkl")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), "--no-python", sys.executable, "-c", WORKER, name, repr(cfgkw), out, backend]
        r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-4000:]
        with open(out, "rb") as f:
            return pickle.load(f)


def run_single(name, cfgkw):
    from paper_2310_07002_b200 import abi, pcv
    from parity_util import Case
    case = Case(name)
    with pcv.Context(0) as c:
        for i, (m, kp, bank) in enumerate(zip(case.models, case.kparams, case.banks)):
            c.add_model(m, kp, bank, model_id=i)
        return c.run(abi.run_config(**cfgkw))


COLUMNS = ["estimate", "log_f_hat", "mc_contribution", "ess", "rhat", "batches", "fault", "failed"]
HEADLINE = ["delta_hat", "mcse", "sigma2_delta", "epistemic_se", "ess_overall", "rhat_max", "verdict_pass",
            "verdict_quantile_value", "iters_run"]


@pytest.mark.parametrize("name,cfgkw", [
    ("cfg1_linreg_loo", dict(chains=4, iters=200, warmup=50, batch_size=20, bench_draws=50, checkpoint_every=100, seed=1)),
    ("ex1_grouped_logo", dict(chains=4, iters=200, warmup=50, batch_size=20, bench_draws=50, seed=2)),
    ("seasonal_hvblock", dict(chains=4, iters=200, warmup=30, batch_size=20, bench_draws=50, checkpoint_every=20,
                              early_stop=1, seed=3)),
])
def test_sharded_bit_identical_to_single(name, cfgkw):
    a = run_sharded(name, cfgkw)
    b = run_single(name, cfgkw)
    for k in COLUMNS:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    np.testing.assert_array_equal(a["divergences"], b["divergences"])
    for k in HEADLINE:
        assert a[k] == b[k] or (np.isnan(a[k]) and np.isnan(b[k])), (k, a[k], b[k])
    np.testing.assert_array_equal(np.sort(a["benchmark"]), np.sort(b["benchmark"]))
    np.testing.assert_array_equal(a["snapshots"], b["snapshots"])


def test_sharded_driver_over_nccl_one_rank():
    """The same driver with the NCCL backend (one rank: NCCL refuses two ranks on one GPU): the
    tensor all-gathers of the fold tables / block sums and the MAX all-reduce run on device buffers,
    and the report equals pcvg_run bit for bit, early stop included."""
    name = "seasonal_hvblock"
    cfgkw = dict(chains=4, iters=200, warmup=30, batch_size=20, bench_draws=50, checkpoint_every=20, early_stop=1,
                 seed=3)
    a = run_sharded(name, cfgkw, world=1, backend="nccl")
    b = run_single(name, cfgkw)
    for k in COLUMNS:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    np.testing.assert_array_equal(a["divergences"], b["divergences"])
    for k in HEADLINE:
        assert a[k] == b[k] or (np.isnan(a[k]) and np.isnan(b[k])), (k, a[k], b[k])
    np.testing.assert_array_equal(a["snapshots"], b["snapshots"])


def test_sharded_logistic_within_rounding_then_mc_error():
    short = dict(chains=4, iters=12, warmup=3, batch_size=3, blocks=4, bench_draws=20, seed=4)
    a, b = run_sharded("logistic_loo", short), run_single("logistic_loo", short)
    rel = np.abs(a["estimate"] - b["estimate"]) / (1 + np.abs(b["estimate"]))
    assert np.mean(rel <= 1e-8) >= 0.9, np.sort(rel)[-5:]
    full = dict(chains=4, iters=100, warmup=20, batch_size=10, bench_draws=50, seed=5)
    a, b = run_sharded("logistic_loo", full), run_single("logistic_loo", full)
    assert abs(a["delta_hat"] - b["delta_hat"]) <= 4 * np.hypot(a["mcse"], b["mcse"])


# ------------------------------------------------------------------------------ in-process multi-device
def run_multi(name, cfgkw, devices):
    from paper_2310_07002_b200 import abi, pcv
    from parity_util import Case
    case = Case(name)
    with pcv.MultiContext(devices) as c:
        for i, (m, kp, bank) in enumerate(zip(case.models, case.kparams, case.banks)):
            c.add_model(m, kp, bank, model_id=i)
        return c.run(abi.run_config(**cfgkw))


@pytest.mark.parametrize("name,cfgkw,devices", [
    ("cfg1_linreg_loo", dict(chains=4, iters=200, warmup=50, batch_size=20, bench_draws=50, checkpoint_every=100, seed=1), [0, 0]),
    ("ex1_grouped_logo", dict(chains=4, iters=200, warmup=50, batch_size=20, bench_draws=50, seed=2), [0, 0, 0]),
    ("seasonal_hvblock", dict(chains=4, iters=200, warmup=30, batch_size=20, bench_draws=50, checkpoint_every=20,
                              early_stop=1, seed=3), [0, 0]),
    ("radon_logo", dict(chains=4, iters=100, warmup=20, batch_size=10, bench_draws=50, seed=4), [0, 0, 0, 0]),
])
def test_multi_device_bit_identical_to_single(name, cfgkw, devices):
    """pcvg_multi_run (csrc/multi_device.cpp: one context per shard, one host thread each, fold-order
    merge) with the shards on cuda:0: every per-fold column, divergence count, benchmark replicate and
    headline statistic equals the single-context pcvg_run bit for bit."""
    a = run_multi(name, cfgkw, devices)
    b = run_single(name, cfgkw)
    for k in COLUMNS:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    np.testing.assert_array_equal(a["divergences"], b["divergences"])
    for k in HEADLINE:
        assert a[k] == b[k] or (np.isnan(a[k]) and np.isnan(b[k])), (k, a[k], b[k])
    np.testing.assert_array_equal(a["benchmark"], b["benchmark"])
    np.testing.assert_array_equal(a["snapshots"], b["snapshots"])
    assert a["gpu_launches"] > 0

"""The FP32 variant of the logistic family (glm32_kernel.cu: tcgen05 kind::tf32 with
hi/lo-split operands): per-step log density and gradient within the north star's FP32 tolerance
of the FP64 oracle (1e-5 relative to the sum of absolute terms), hmc steps and end-to-end elpd
within Monte Carlo error of the FP64 path."""
import numpy as np
import pytest

from paper_2310_07002_b200 import abi, pcv
import _oracle as O
from parity_util import Case, sample_thetas, term_scales

pytestmark = pytest.mark.gpu

RTOL32 = 1e-5


@pytest.fixture(scope="module")
def case():
    return Case("logistic_loo")


def ctx_tf32(case):
    c = pcv.Context(0)
    c.set_kernel_policy(c.KERNEL_TF32)
    slot = c.add_model(case.models[0], case.kparams[0], case.banks[0], model_id=0)
    return c, slot


def test_tf32_log_joint_and_gradient(case):
    c, slot = ctx_tf32(case)
    om = case.omodels[0]
    worst = 0.0
    for fold in (0, 1, case.K // 2, case.K - 1, case.K):
        th = sample_thetas(case, 0, 6, seed=fold)
        lp, g = c.eval(slot, np.full(len(th), fold), th)
        for i in range(len(th)):
            s_lp, s_g = term_scales(case, 0, th[i], fold)
            e1 = abs(lp[i] - om.log_joint(th[i], fold)) / s_lp
            e2 = np.abs(g[i] - om.grad(th[i], fold)).max() / s_g
            worst = max(worst, e1, e2)
            assert e1 <= RTOL32 and e2 <= RTOL32, (fold, e1, e2)
    print(f"tf32 worst scaled error {worst:.2e}")
    c.close()


def test_tf32_hmc_step(case):
    c, slot = ctx_tf32(case)
    om, kp = case.omodels[0], case.kparams[0]
    rng = np.random.default_rng(3)
    th = sample_thetas(case, 0, 8, seed=5)
    folds = rng.integers(0, case.K + 1, 8).astype(np.int32)
    mom = rng.standard_normal(th.shape) / np.sqrt(kp.inv_mass_diag)
    u = rng.uniform(size=8)
    out, h0, h1, acc, div = c.hmc_probe(slot, folds, th, mom, u)
    for i in range(8):
        oth, oh0, oh1, oacc, odiv = om.hmc_probe(int(folds[i]), kp.step_size, kp.n_leapfrog, kp.inv_mass_diag,
                                                 th[i], mom[i], u[i])
        s_lp, _ = term_scales(case, 0, th[i], int(folds[i]))
        assert abs(h0[i] - oh0) <= RTOL32 * s_lp and abs(h1[i] - oh1) <= 1e-4 * s_lp
        np.testing.assert_allclose(out[i], oth, rtol=1e-3, atol=1e-3)
    c.close()


def test_tf32_run_within_mc_error(case):
    c, slot = ctx_tf32(case)
    rc = case.z["run_cfg"]
    cfg = abi.run_config(chains=int(rc[0]), iters=int(rc[1]), warmup=int(rc[2]), batch_size=int(rc[3]),
                         bench_draws=int(rc[5]), seed=1)
    rep = c.run(cfg)
    c.close()
    ref = float(case.z["ref_delta_hat"])
    tol = 4.0 * np.hypot(rep["mcse"], float(case.z["ref_mcse"])) + 1e-6
    assert abs(rep["delta_hat"] - ref) <= tol, (rep["delta_hat"], ref, tol)
    assert np.isfinite(rep["rhat_max"])


def _run_sub(code, env):
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=900, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    return r.stdout


def test_tf32_row_split_cluster_matches_oracle():
    """Row-split clusters (glm32_kernel cs > 1, the wave-tail path) forced on every tile: log joint,
    gradient and injected-momentum hmc_step within the FP32 tolerance of the FP64 oracle."""
    code = r'''
import sys, numpy as np
sys.path[:0] = ["tests", "tests/golden", "."]
from parity_util import Case, sample_thetas, term_scales
from paper_2310_07002_b200 import pcv
case = Case("logistic_loo"); om, kp = case.omodels[0], case.kparams[0]
c = pcv.Context(0); c.set_kernel_policy(c.KERNEL_TF32)
slot = c.add_model(case.models[0], kp, case.banks[0], model_id=0)
worst = 0.0
for fold in (0, 1, case.K // 2, case.K):
    th = sample_thetas(case, 0, 6, seed=fold)
    lp, g = c.eval(slot, np.full(len(th), fold), th)
    for i in range(len(th)):
        s_lp, s_g = term_scales(case, 0, th[i], fold)
        worst = max(worst, abs(lp[i] - om.log_joint(th[i], fold)) / s_lp, np.abs(g[i] - om.grad(th[i], fold)).max() / s_g)
rng = np.random.default_rng(3)
th = sample_thetas(case, 0, 8, seed=5)
folds = rng.integers(0, case.K + 1, 8).astype(np.int32)
mom = rng.standard_normal(th.shape) / np.sqrt(kp.inv_mass_diag)
u = rng.uniform(size=8)
out, h0, h1, acc, div = c.hmc_probe(slot, folds, th, mom, u)
hworst = 0.0
for i in range(8):
    oth, oh0, oh1, oacc, odiv = om.hmc_probe(int(folds[i]), kp.step_size, kp.n_leapfrog, kp.inv_mass_diag, th[i], mom[i], u[i])
    s_lp, _ = term_scales(case, 0, th[i], int(folds[i]))
    hworst = max(hworst, abs(h0[i] - oh0) / s_lp, abs(h1[i] - oh1) / s_lp / 10)
    np.testing.assert_allclose(out[i], oth, rtol=1e-3, atol=1e-3)
print(worst, hworst)
'''
    worst, hworst = map(float, _run_sub(code, {"PCVG_GLM32_CS": "4"}).split()[-2:])
    assert worst <= RTOL32 and hworst <= RTOL32, (worst, hworst)


def test_tf32_wave_tail_split_matches_unsplit():
    """More than one wave of 128-chain tiles: the last partial wave runs as row-split clusters.
    Chains of the full waves are bit-identical to an unsplit launch; tail chains differ only by the
    FP32 summation grouping of G, so their fold estimates agree to MC-irrelevant precision."""
    code = r'''
import sys, numpy as np
sys.path[:0] = ["tests", "tests/golden", "."]
from parity_util import Case
from paper_2310_07002_b200 import abi, pcv
case = Case("logistic_loo")
with pcv.Context(0) as c:
    c.set_kernel_policy(c.KERNEL_TF32)
    c.add_model(case.models[0], case.kparams[0], case.banks[0], model_id=0)
    rep = c.run(abi.run_config(chains=40, iters=6, warmup=2, batch_size=3, bench_draws=5, seed=2))
np.save(sys.argv[1] if len(sys.argv) > 1 else "/tmp/x.npy", rep["estimate"])
print(" ".join(repr(float(v)) for v in rep["estimate"]))
'''
    out = {}
    for tag, env in (("split", {}), ("plain", {"PCVG_NO_TAIL_SPLIT": "1"})):
        out[tag] = np.array([float(v) for v in _run_sub(code, env).split()])
    a, b = out["split"], out["plain"]
    assert a.shape == (500,)  # 500 folds x 40 chains = 157 tiles of 128: 148 + a 9-tile tail
    full = 148 * 128 // 40  # folds entirely in the full waves
    assert np.all(a[:full] == b[:full])
    rel = np.abs(a[full:] - b[full:]) / (1.0 + np.abs(b[full:]))
    assert np.all(np.isfinite(a)) and np.median(rel) <= 1e-3, np.sort(rel)[-5:]

"""GPU parity at the HBM-streaming size of the logistic path: N = 400,000, P = 50, so the padded
design matrix (166 MB) no longer fits the 126 MB L2 and every pass streams X tiles from HBM
through the TMA ring (parity_util.StreamCase; the throughput and ncu evidence come from
tools/bench_streaming.py). Same probes and tolerances as the cfg2 bench shape
(test_gpu_bench_shapes.py): log joint, gradient and log_pred, and leapfrog end points with one
gradient-only (fast-sigmoid) pass, at 1e-12 of the sum of absolute terms, for a full wave plus
a wave tail and for a single 64-chain tile split over several clusters."""
import numpy as np
import pytest

from parity_util import StreamCase
from test_gpu_bench_shapes import RTOL, context, logistic_scales, one_tile_points, wave_and_tail_points

pytestmark = pytest.mark.gpu

_case = []


def stream_case():
    if not _case:
        _case.append(StreamCase())
    return _case[0]


def _thin(check, n):
    """At most n checked chains (the oracle's log joint costs 20M flops at this size)."""
    if len(check) <= n:
        return check
    return np.concatenate([check[:4], np.random.default_rng(0).choice(check[4:], n - 4, replace=False)])


@pytest.mark.parametrize("geometry", ["wave+tail", "one-tile-cluster"])
def test_streaming_log_joint_gradient_and_log_pred(geometry):
    cs = stream_case()
    om = cs.omodels[0]
    th, folds, check = (wave_and_tail_points if geometry == "wave+tail" else one_tile_points)(cs, 31)
    check = _thin(check, 40)
    c, (slot,) = context(cs)
    lp, g = c.eval(slot, folds, th)
    pred = c.eval_pred(slot, folds, th)
    c.close()
    for i in check:
        f = int(folds[i])
        s_lp, s_g = logistic_scales(cs, th[i], f)
        olp, og = om.log_joint(th[i], f), om.grad(th[i], f)
        assert abs(lp[i] - olp) <= RTOL * s_lp, (i, f, lp[i], olp, s_lp)
        err = np.abs(g[i] - og) / s_g
        assert err.max() <= RTOL, (i, f, err.max(), int(err.argmax()))
        opred = om.log_pred(th[i], f)
        assert abs(pred[i] - opred) <= RTOL * (1.0 + abs(np.sum(opred))), (i, f, pred[i], opred)


@pytest.mark.parametrize("geometry", ["wave+tail", "one-tile-cluster"])
def test_streaming_leapfrog_two_steps(geometry):
    cs = stream_case()
    om, kp = cs.omodels[0], cs.kparams[0]
    th, folds, check = (wave_and_tail_points if geometry == "wave+tail" else one_tile_points)(cs, 32)
    check = _thin(check, 24)
    rng = np.random.default_rng(33)
    mom = rng.standard_normal(th.shape) / np.sqrt(kp.inv_mass_diag)
    c, (slot,) = context(cs, n_lf=2)
    q1, p1, ok = c.leapfrog(slot, folds, th, mom)
    c.close()
    eps, im = kp.step_size, kp.inv_mass_diag
    for i in check:
        f = int(folds[i])
        okr, oq, op = om.leapfrog(f, eps, 2, im, th[i], mom[i])
        assert bool(ok[i]) == bool(okr), (i, f)
        if not okr:
            continue
        _, s_g0 = logistic_scales(cs, th[i], f)
        _, s_g1 = logistic_scales(cs, oq, f)
        s_p = np.abs(mom[i]) + eps * 2 * np.maximum(s_g0, s_g1)
        s_q = np.abs(th[i]) + eps * 2 * im * s_p
        assert (np.abs(p1[i] - op) / s_p).max() <= RTOL and (np.abs(q1[i] - oq) / s_q).max() <= RTOL, (i, f)

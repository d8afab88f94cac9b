"""CPU check of the gradient-pass logistic residual's arithmetic (tc_common.cuh::logistic_resid_fast).

The kernel computes y - sigmoid(x) with a table + degree-4 polynomial e^-|x|, integer exponent
assembly, one FMA for 1 + e^-|x|, and a shared reciprocal for both signs of x. This restates each
step in float64 numpy (the hardware rcp.approx is modelled as 1/d rounded to 22 bits, its stated
accuracy, followed by the kernel's Newton step) and compares with the exact residual in long double.
Bound: absolute error <= 1e-13 on the residual (4.7e-14 measured), far inside the per-step gradient tolerance
(1e-12 * sum|terms|); the reference computes sigmoid with std::exp (model.hpp:24-78
conventions for the logistic plugin).
"""
import numpy as np

from tools.exp_poly import coefficients, max_rel_error

C1, C2, C3, C4 = 0.9999999999641696, 0.4999999999940276, 0.1666678885252701, 0.04166687031843588


def _fma(a, b, c):
    ld = np.longdouble
    return (ld(a) * ld(b) + ld(c)).astype(np.float64)


def _resid_fast(x, y):
    x = np.asarray(x, dtype=np.float64)
    bits = x.view(np.int64)
    xh = (bits >> 32).astype(np.int32)
    ah = xh & 0x7FFFFFFF
    absx = np.abs(x)
    a = np.where(ah >= 0x4085E000, 700.0, absx)
    shift = 6755399441055744.0
    t = _fma(a, 46.16624130844683, shift)
    n = (t.view(np.int64) & 0xFFFFFFFF).astype(np.int64)
    nd = t - shift
    r = _fma(nd, 0.02166084939249829, -a)
    p = _fma(r, C4, C3)
    p = _fma(p, r, C2)
    p = _fma(p, r, C1)
    p = _fma(p, r, 1.0)
    tab = np.exp2(-np.arange(32) / 32.0)
    tv = tab[n & 31]
    scaled = (tv.view(np.int64) - ((n >> 5) << 52)).view(np.float64)
    d = _fma(scaled, p, 1.0)
    r0 = 1.0 / d
    m, e = np.frexp(r0)
    r0 = np.ldexp(np.round(m * 2.0**22) / 2.0**22, e)  # rcp.approx.ftz.f64 ~ 2^-22
    err = _fma(-d, r0, 1.0)
    inv = _fma(r0, err, r0)
    pos = xh >= 0
    return _fma(np.where(pos, -1.0, 1.0), inv, np.where(pos, y, y - 1.0))


def _resid_exact(x, y):
    ld = np.longdouble
    xl = np.asarray(x).astype(ld)
    with np.errstate(over="ignore"):
        return (np.asarray(y).astype(ld) - ld(1) / (ld(1) + np.exp(-xl))).astype(np.float64)


def test_poly_coefficients_and_error():
    c, R = coefficients()
    assert c[0] == 1.0
    assert [c[1], c[2], c[3], c[4]] == [C1, C2, C3, C4]
    assert max_rel_error(c, R) < 1e-13


def test_residual_matches_exact_sigmoid():
    rng = np.random.default_rng(3)
    x = np.concatenate([
        rng.normal(0, 1, 20000), rng.normal(0, 8, 20000), rng.uniform(-40, 40, 20000),
        np.array([0.0, -0.0, 1e-300, -1e-300, 699.9, 700.0, 700.1, -700.1, 1e5, -1e5, 36.7, -36.7]),
    ])
    for y in (0.0, 1.0):
        got = _resid_fast(x, y)
        want = _resid_exact(x, y)
        assert np.all(np.isfinite(got))
        assert np.max(np.abs(got - want)) < 1e-13  # measured 4.7e-14, dominated by the reciprocal


def test_signed_zero_and_nan_are_finite():
    got = _resid_fast(np.array([0.0, -0.0]), 1.0)
    assert np.allclose(got, 0.5, rtol=0, atol=1e-15)
    # NaN clamps to |x| = 700 exactly as fmin(NaN, 700) does: a finite residual, as before
    assert np.all(np.isfinite(_resid_fast(np.array([np.nan]), 0.0)))

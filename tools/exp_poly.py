"""Coefficients of the degree-4 polynomial for e^r on |r| <= ln2/64 used by
tc_common.cuh::logistic_resid_fast: interpolation at the 5 Chebyshev nodes (near-minimax),
solved in long double, rounded to double, and the relative error measured on a dense grid.
"""
import numpy as np

ld = np.longdouble


def coefficients(deg=4, half_width=None):
    R = half_width if half_width is not None else np.log(ld(2)) / ld(64)
    k = np.arange(deg + 1)
    nodes = np.cos((2 * k + 1) * np.pi / (2 * (deg + 1))).astype(ld) * R
    M = [[n ** j for j in range(deg + 1)] + [np.exp(n)] for n in nodes]
    for i in range(deg + 1):
        for r in range(i + 1, deg + 1):
            f = M[r][i] / M[i][i]
            M[r] = [a - f * b for a, b in zip(M[r], M[i])]
    c = [ld(0)] * (deg + 1)
    for i in reversed(range(deg + 1)):
        c[i] = (M[i][deg + 1] - sum(M[i][j] * c[j] for j in range(i + 1, deg + 1))) / M[i][i]
    return [float(x) for x in c], R


def max_rel_error(c, R, n=200001):
    rs = np.linspace(-float(R), float(R), n).astype(ld)
    p = ld(c[-1])
    for cj in reversed(c[:-1]):
        p = p * rs + ld(cj)
    return float(np.max(np.abs(p / np.exp(rs) - 1)))


if __name__ == "__main__":
    c, R = coefficients()
    print("coefficients c0..c4:", [repr(x) for x in c])
    print("max relative error on |r| <= ln2/64:", max_rel_error(c, R))

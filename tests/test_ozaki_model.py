"""CPU model of reading R10: the fp64 product U = M W computed as exact integer sums of
int8 slice products (the arithmetic k_oz_symm runs on the INT8 tensor cores), checked against EXACT rational
arithmetic.  It pins the two claims the GPU path rests on:
  * with the D scaling of an SPD M every scaled entry is below 4 in magnitude (one scale per block suffices),
    and every int8 digit / int32 diagonal sum stays in range;
  * the result is within the stated bound of the exact product: |U - M W| <= 2^-53 |MW| + b 2^-54 sigma mu
    per entry (representation of each scaled entry to 2^-56 of its scale, the dropped diagonals i + j >= 7,
    the final rounding) - i.e. as accurate as an fp64 product.
This is a model written from the reading, not from the CUDA source; it shares no code with it."""
from fractions import Fraction
import math

import numpy as np
import pytest


def digits(x):
    """X = rint(x 2^55), |x| < 1/2, as 7 signed base-256 digits, most significant first."""
    X = int(round(x * 2.0 ** 55))      # exact: x * 2^55 is an exact double; round() = rint (ties to even)
    d = []
    for _ in range(6):
        lo = ((X & 0xFF) ^ 0x80) - 0x80  # signed low byte
        d.append(lo)
        X = (X - lo) >> 8
    d.append(X)
    return d[::-1], X


def exp_above(m):
    return math.frexp(m)[1] if m > 0 else 0


def ozaki_product(M, W):
    """U = M W by the R10 splitting (Python integers: exact int32 sums, checked for range)."""
    b, s = W.shape
    e = np.array([math.floor((math.frexp(M[n, n])[1] - 1) / 2) for n in range(b)])   # D = 2^e
    Mt = M / np.ldexp(1.0, e)[:, None] / np.ldexp(1.0, e)[None, :]
    assert np.abs(Mt).max() < 4.0          # Mt_nn in [1, 4), |Mt_kn| <= sqrt(Mt_kk Mt_nn) < 4 for SPD M
    mu = exp_above(np.abs(Mt).max()) + 1
    Wt = W * np.ldexp(1.0, e)[:, None]
    sig = [exp_above(np.abs(Wt[:, c]).max()) + 1 for c in range(s)]
    dM = [[digits(math.ldexp(Mt[k, n], -mu))[0] for n in range(b)] for k in range(b)]
    dW = [[digits(math.ldexp(Wt[k, c], -sig[c]))[0] for c in range(s)] for k in range(b)]
    for k in range(b):
        for n in range(b):
            assert abs(dM[k][n][0]) <= 64 and all(-128 <= v <= 127 for v in dM[k][n])
    U = np.empty((b, s))
    for n in range(b):
        for c in range(s):
            acc = [0] * 7
            for i in range(7):
                for j in range(7 - i):
                    acc[i + j] += sum(dW[k][c][i] * dM[k][n][j] for k in range(b))
            assert all(abs(a) < 2 ** 31 for a in acc)               # int32 accumulators
            hi = (acc[0] << 16) + (acc[1] << 8) + acc[2]
            lo = (acc[3] << 24) + (acc[4] << 16) + (acc[5] << 8) + acc[6]
            u = math.fma(float(hi), 2.0 ** -30, float(lo) * 2.0 ** -62) if hasattr(math, "fma") else \
                float(hi) * 2.0 ** -30 + float(lo) * 2.0 ** -62
            U[n, c] = math.ldexp(u, sig[c] + mu + int(e[n]))
    return U, sig, mu


def _spd(b, rng, spread):
    Q, _ = np.linalg.qr(rng.standard_normal((b, b)))
    lam = np.exp(rng.uniform(-spread, spread, b))
    M = (Q * lam) @ Q.T
    return (M + M.T) / 2


@pytest.mark.parametrize("b,s,spread,wscale", [(24, 3, 1.0, 1.0), (40, 2, 6.0, 1e-3), (33, 4, 3.0, 1e120)])
def test_ozaki_model_matches_exact_product(b, s, spread, wscale):
    rng = np.random.default_rng(b)
    M = _spd(b, rng, spread)
    D = np.exp(rng.uniform(-4, 4, b))           # badly scaled rows / columns (S_j^-1 of a graded mesh)
    M = D[:, None] * M * D[None, :]
    W = rng.standard_normal((b, s)) * wscale
    W[:, 0] *= 1e-9                               # columns of very different size
    U, sig, mu = ozaki_product(M, W)
    for n in range(b):
        for c in range(s):
            exact = sum(Fraction(M[n, k]) * Fraction(W[k, c]) for k in range(b))
            absdot = sum(abs(Fraction(M[n, k]) * Fraction(W[k, c])) for k in range(b))
            err = abs(Fraction(U[n, c]) - exact)
            # fp64-level bound: final rounding + per-entry representation / dropped diagonals relative to the
            # row's scaled magnitude (delta_n sigma_c mu: the scale the fixed-point digits are taken against)
            e_n = math.floor((math.frexp(M[n, n])[1] - 1) / 2)
            scale = Fraction(2) ** (sig[c] + mu + e_n)
            bound = Fraction(2) ** -53 * abs(exact) + b * Fraction(2) ** -54 * scale
            assert err <= bound, (n, c, float(err), float(bound))
            # and never worse than a few units of an fp64 dot product's own worst-case error bound
            assert err <= 4 * b * Fraction(2) ** -53 * absdot + Fraction(2) ** -53 * abs(exact) + \
                b * Fraction(2) ** -54 * scale


def test_ozaki_model_zero_and_identity():
    b = 8
    M = np.eye(b) * 3.0
    W = np.zeros((b, 2))
    W[:, 1] = np.arange(1, b + 1)
    U, _, _ = ozaki_product(M, W)
    assert np.all(U[:, 0] == 0)
    assert np.array_equal(U[:, 1], 3.0 * W[:, 1])   # exact when every product is exact

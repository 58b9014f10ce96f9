"""Independent reference routines used by the oracle pin tests.

These re-derive results from textbook definitions WITHOUT calling the oracle
(carry-less polynomial products for GF(2^m), Sylvester-Hadamard matrices from
scipy, brute-force codeword enumeration), so a mistake in the oracle cannot
hide behind itself.
"""
import itertools

import numpy as np
import scipy.linalg

DEFAULT_POLY = {1: 0x3, 2: 0x7, 3: 0xB, 4: 0x13, 5: 0x25, 6: 0x43, 7: 0x89, 8: 0x11D}


def clmul_mod(a: int, b: int, m: int, poly: int) -> int:
    """Product in GF(2)[x]/(poly): carry-less multiply then reduce."""
    r = 0
    for i in range(m):
        if (b >> i) & 1:
            r ^= a << i
    for d in range(2 * m - 2, m - 1, -1):
        if (r >> d) & 1:
            r ^= poly << (d - m)
    return r


def hadamard(m: int) -> np.ndarray:
    """Sylvester Hadamard matrix; entry [z, x] = (-1)^{popcount(z & x)}."""
    return scipy.linalg.hadamard(1 << m).astype(np.float64)


def bit_prior(llr: np.ndarray) -> np.ndarray:
    """p(x) = prod_i Pr(b_i = x_i) for independent bits, Pr(b=0) = 1/(1+e^-L)."""
    m = len(llr)
    q = 1 << m
    p = np.ones(q)
    for x in range(q):
        for i in range(m):
            L = llr[i]
            p[x] *= 1 / (1 + np.exp(L)) if (x >> i) & 1 else 1 / (1 + np.exp(-L))
    return p


def enumerate_codewords(M, N, m, poly, rows, cols, coeffs):
    """All x in GF(2^m)^N with H x = 0, by exhaustive search (tiny codes only)."""
    q = 1 << m
    mul = np.array([[clmul_mod(a, b, m, poly) for b in range(q)] for a in range(q)], dtype=np.int64)
    X = np.array(list(itertools.product(range(q), repeat=N)), dtype=np.int64)
    ok = np.ones(len(X), bool)
    for c in range(M):
        s = np.zeros(len(X), np.int64)
        for r, v, h in zip(rows, cols, coeffs):
            if r == c:
                s ^= mul[h, X[:, v]]
        ok &= s == 0
    return X[ok]

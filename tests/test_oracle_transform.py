"""Pins for the oracle's transforms."""
import numpy as np
import pytest

import oracle
from conftest import golden_lines
from helpers import bit_prior, hadamard


@pytest.mark.parametrize("m", [1, 2, 3, 5, 8])
def test_wht_equals_hadamard_matrix(m):
    rng = np.random.default_rng(m)
    p = rng.random(1 << m)
    np.testing.assert_allclose(oracle.wht(p), hadamard(m) @ p, rtol=1e-13, atol=1e-13)
    # involution: WHT(WHT(p)) = 2^m p; iwht inverts
    np.testing.assert_allclose(oracle.wht(oracle.wht(p)), (1 << m) * p, rtol=1e-12)
    np.testing.assert_allclose(oracle.iwht(oracle.wht(p)), p, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("m", [1, 2, 4, 6])
def test_convolution_theorem(m):
    # WHT(p1 (x) p2) = WHT(p1) WHT(p2) pointwise
    rng = np.random.default_rng(100 + m)
    a, b = rng.random(1 << m), rng.random(1 << m)
    a /= a.sum()
    b /= b.sum()
    Hd = hadamard(m)
    np.testing.assert_allclose(Hd @ oracle.convolve(a, b), (Hd @ a) * (Hd @ b), rtol=1e-12, atol=1e-14)


def test_spec_examples():
    for row in golden_lines("spec_transform_examples.txt"):
        kind, vals = row[0], [float(v) for v in row[1:]]
        if kind == "conv":
            np.testing.assert_allclose(oracle.convolve(vals[0:2], vals[2:4]), vals[4:6], atol=1e-15)
        elif kind == "boxplus":
            s1, l1 = oracle.gamma(vals[0:2])
            s2, l2 = oracle.gamma(vals[2:4])
            so, lo = oracle.boxplus(s1, l1, s2, l2)
            np.testing.assert_allclose(oracle.gamma_inv(so, lo), vals[4:6], atol=1e-15)
        elif kind == "wht":
            np.testing.assert_allclose(oracle.wht(vals[0:2]), vals[2:4], atol=0)
        elif kind == "iwht":
            np.testing.assert_allclose(oracle.iwht(vals[0:2]), vals[2:4], atol=0)
        elif kind == "gamma":
            s, l = oracle.gamma([vals[0]])
            assert int(s[0]) == int(vals[1])
            assert abs(l[0] - vals[2]) < 1e-15
        elif kind == "spmap":
            # single check H = [1 1] over GF(2): SP posterior of v1 after one iteration
            f = oracle.Field(1, 0x3)
            code = oracle.Code(f, 1, 2, [0, 0], [0, 1], [1, 1])
            p0 = np.array([vals[0:2], vals[2:4]])
            w = code.sp_check_to_variable(code.sp_variable_to_check(p0, np.ones((2, 2))))
            qv = code.sp_posterior(p0, w)
            ref = np.array(vals[4:6]) / sum(vals[4:6])
            np.testing.assert_allclose(qv[0], ref, rtol=1e-12)


def test_gamma_homomorphism():
    # Gamma(xy) = Gamma(x) + Gamma(y) (GF(2) sum of signs, real sum of logs)
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, 10000)
    y = rng.uniform(-1, 1, 10000)
    sx, lx = oracle.gamma(x)
    sy, ly = oracle.gamma(y)
    sp, lp = oracle.gamma(x * y)
    assert np.array_equal(sp, sx ^ sy)
    np.testing.assert_allclose(lp, lx + ly, rtol=0, atol=1e-12)


@pytest.mark.parametrize("m", [2, 3, 6])
def test_boxplus_is_signed_xor_convolution(m):
    # Gamma^{-1}(A [+] B)(z) = sum_y A(y) B(z^y); checked through the convolution
    # theorem with scipy Hadamard matrices: A [+] B = H^{-1}( (H A) * (H B) ).
    rng = np.random.default_rng(200 + m)
    q = 1 << m
    a, b = rng.uniform(-1, 1, q), rng.uniform(-1, 1, q)
    a[0] = b[0] = 1.0
    sa, la = oracle.gamma(a)
    sb, lb = oracle.gamma(b)
    so, lo = oracle.boxplus(sa, la, sb, lb)
    Hd = hadamard(m)
    ref = (Hd @ ((Hd @ a) * (Hd @ b))) / q
    np.testing.assert_allclose(oracle.gamma_inv(so, lo), ref, rtol=1e-11, atol=1e-13)


@pytest.mark.parametrize("m", [2, 4, 6, 8])
def test_lf_init_is_tanh_product_closed_form(m):
    # INIT Lambda^(0) = Gamma(WHT(p^(0))) equals the closed form
    # P^(0)(z) = prod_{i: z_i=1} tanh(L_i/2) (Gallager's f).
    rng = np.random.default_rng(300 + m)
    N = 5
    f = oracle.Field(m, {2: 0x7, 4: 0x13, 6: 0x43, 8: 0x11D}[m])
    code = oracle.Code(f, 1, N, [0] * N, list(range(N)), [1] * N)
    llr = rng.normal(2.5, 2.2, N * m)
    S0, L0 = code.lf_init(llr)
    q = 1 << m
    for v in range(N):
        t = np.tanh(llr[v * m:(v + 1) * m] / 2)
        P = np.array([np.prod([t[i] for i in range(m) if (z >> i) & 1]) for z in range(q)])
        lin = np.where(S0[v] == 1, -1.0, 1.0) * np.exp(L0[v])
        np.testing.assert_allclose(lin, P, rtol=1e-9, atol=1e-15)
        # and the oracle prior is the factorised posterior (independent route)
        np.testing.assert_allclose(oracle.channel_prior(llr[v * m:(v + 1) * m]), bit_prior(llr[v * m:(v + 1) * m]),
                                   rtol=1e-13)

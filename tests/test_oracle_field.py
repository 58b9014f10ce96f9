"""Pins for the oracle's GF(2^m) layer (Appendix A :656-680)."""
import numpy as np
import pytest

import oracle
from helpers import DEFAULT_POLY, clmul_mod, hadamard
from conftest import golden_lines


def test_gf8_matches_paper_listing():
    # the worked GF(8) example, alpha^3 + alpha + 1 = 0.
    f = oracle.Field(3, 0b1011)
    for row in golden_lines("gf8_paper_listing.txt"):
        i, bits = int(row[0]), [int(b) for b in row[1:]]
        val = f.exp(i)
        assert [(val >> r) & 1 for r in range(3)] == bits
        assert f.log(val) == i


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6, 7, 8])
def test_gf_mul_equals_carryless_product(m):
    f = oracle.Field(m, DEFAULT_POLY[m])
    q = 1 << m
    rng = np.random.default_rng(m)
    pairs = [(a, b) for a in range(q) for b in range(q)] if q <= 64 else [tuple(rng.integers(0, q, 2)) for _ in range(4000)]
    for a, b in pairs:
        assert f.mul(a, b) == clmul_mod(int(a), int(b), m, DEFAULT_POLY[m])
    for a in range(1, q):
        assert f.mul(a, f.inv(a)) == 1


@pytest.mark.parametrize("m", [2, 3, 4])
def test_distributivity_exhaustive(m):
    f = oracle.Field(m, DEFAULT_POLY[m])
    q = 1 << m
    for a in range(q):
        for b in range(q):
            for c in range(q):
                assert f.mul(a, b ^ c) == f.mul(a, b) ^ f.mul(a, c)


def test_non_primitive_rejected():
    with pytest.raises(ValueError):
        oracle.Field(3, 0b1111)      # x^3+x^2+x+1 reducible
    with pytest.raises(ValueError):
        oracle.Field(4, 0b11111)     # x^4+x^3+x^2+x+1 irreducible, period 5
    with pytest.raises(ValueError):
        oracle.Field(3, 0b111)       # wrong degree


@pytest.mark.parametrize("m", [2, 3, 4, 6, 8])
def test_companion_power_multiplies_by_alpha_power(m):
    # A^i alpha^j = alpha^{i+j}; the oracle stores (A^i)^T (:672).
    f = oracle.Field(m, DEFAULT_POLY[m])
    q = 1 << m
    for i in range(0, q - 1, max(1, (q - 1) // 17)):
        Ai = f.companion_pow_T(i).T.copy()
        for j in range(q - 1):
            assert f.apply_binary_matrix(Ai, f.exp(j)) == f.exp(i + j)


def test_dot_parity_paper_example():
    rows = {r[0]: r[1:] for r in golden_lines("dot_parity_paper_example.txt")}
    z = sum(int(b) << i for i, b in enumerate(rows["z"]))
    x = sum(int(b) << i for i, b in enumerate(rows["x"]))
    assert bin(z & x).count("1") == int(rows["dot"][0])
    assert oracle.dot_parity(z, x) == int(rows["dot"][0]) % 2


def _appendix_sides(f, h, p):
    # LHS: FT of p~(x) = p(h^{-1} x)
    # RHS: P(H_cv z)
    m, q = f.m, f.q
    hinv = f.inv(h)
    ptil = np.array([p[f.mul(hinv, x)] for x in range(q)])
    Hd = hadamard(m)
    lhs = Hd @ ptil
    P = Hd @ p
    rhs = np.array([P[f.fourier_perm(h, z)] for z in range(q)])
    field_mult = np.array([P[f.mul(h, z)] for z in range(q)])
    return lhs, rhs, field_mult


@pytest.mark.parametrize("m,nh", [(2, None), (3, None), (4, None), (6, 20), (8, 12)])
def test_appendix_permutation_lemma(m, nh):
    # Appendix A for every h (m <= 4) or sampled h (m = 6, 8).
    f = oracle.Field(m, DEFAULT_POLY[m])
    q = 1 << m
    rng = np.random.default_rng(10 + m)
    hs = range(1, q) if nh is None else rng.integers(1, q, nh)
    transpose_bug_detected = False
    for h in hs:
        p = rng.random(q)
        p /= p.sum()
        lhs, rhs, fm = _appendix_sides(f, int(h), p)
        np.testing.assert_allclose(lhs, rhs, rtol=0, atol=1e-13)
        if not np.allclose(lhs, fm):
            transpose_bug_detected = True
    # For m >= 3 indexing by the field product h*z (i.e. M_h instead of M_h^T) is wrong
    # for some h; GF(4) cannot tell the two apart (all M_h symmetric, SURVEY finding 1).
    assert transpose_bug_detected == (m >= 3)


@pytest.mark.parametrize("m", [3, 6])
def test_fourier_perm_is_linear_bijection(m):
    f = oracle.Field(m, DEFAULT_POLY[m])
    q = 1 << m
    for h in range(1, q):
        img = [f.fourier_perm(h, z) for z in range(q)]
        assert sorted(img) == list(range(q))
        for a in range(0, q, 3):
            for b in range(0, q, 5):
                assert img[a ^ b] == img[a] ^ img[b]
        for z in range(q):
            assert f.fourier_perm_inv(h, img[z]) == z
            # inverse permutation is the permutation of h^{-1}
            assert f.fourier_perm(f.inv(h), img[z]) == z

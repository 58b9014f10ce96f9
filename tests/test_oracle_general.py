"""Pins for the oracle's Log-Fourier SP at column weights j != 2.

O-LF's node rules are written for any |C_v|, so the pins of the j = 2 case
extend: per-edge, per-iteration agreement with the probability-domain O-SP on (3,k)- and
(4,k)-regular and mixed-weight codes, and the symbol posterior equal to O-SP's.  (Weight-1 leaves
are already exercised by the exact-on-trees pins of test_oracle_decoder.py.)"""
import numpy as np
import pytest

import oracle
import synth
from helpers import DEFAULT_POLY, hadamard


def _agree(code, llr, iters):
    Hd = hadamard(code.m)
    _, ecol, _ = code.edges()
    p0 = code.sp_init(llr)
    S0, L0 = code.lf_init(llr)
    u, Us, Ul = p0[ecol].copy(), S0[ecol].copy(), L0[ecol].copy()
    for _ in range(iters):
        w = code.sp_check_to_variable(u)
        Ws, Wl = code.lf_check_to_variable(Us, Ul)
        Wsp = w @ Hd.T
        Wsp /= Wsp[:, :1]
        np.testing.assert_allclose(np.where(Ws, -1, 1) * np.exp(Wl), Wsp, rtol=1e-9, atol=1e-9)
        u = code.sp_variable_to_check(p0, w)
        Us, Ul, ev = code.lf_variable_to_check(S0, L0, Ws, Wl)
        assert ev == 0
        np.testing.assert_allclose(np.where(Us, -1, 1) * np.exp(Ul), u @ Hd.T, rtol=1e-9, atol=1e-9)
        post, _ = code.lf_symbol_posterior(S0, L0, Ws, Wl)
        np.testing.assert_allclose(post, code.sp_posterior(p0, w), rtol=1e-8, atol=1e-12)


@pytest.mark.parametrize("m,N,k,j,seed", [(3, 16, 6, 3, 101), (2, 24, 6, 3, 102), (4, 12, 6, 4, 103), (5, 8, 6, 3, 104)])
def test_lf_equals_sp_at_higher_column_weight(m, N, k, j, seed):
    M, rows, cols, coeffs = synth.make_regular_code(N, k, m, seed, j=j)
    code = oracle.Code(oracle.Field(m, DEFAULT_POLY[m]), M, N, rows, cols, coeffs)
    llr = np.random.default_rng(seed).normal(1.0, 1.8, N * m)
    _agree(code, llr, 4)


def test_lf_equals_sp_mixed_column_weights():
    # weights 1, 2, 3 mixed: a (2,k) code plus extra rows over some variables, minus one edge
    m, N, k = 3, 16, 4
    M, rows, cols, coeffs = synth.make_regular_code(N, k, m, 111)
    rng = np.random.default_rng(111)
    extra_v = rng.choice(N, 6, replace=False)
    rows = np.concatenate([rows, np.full(3, M), np.full(3, M + 1)])
    cols = np.concatenate([cols, extra_v])
    coeffs = np.concatenate([coeffs, rng.integers(1, 8, 6)])
    drop = np.where(cols == np.setdiff1d(np.arange(N), extra_v)[0])[0][0]
    keep = np.ones(len(rows), bool)
    keep[drop] = False
    code = oracle.Code(oracle.Field(m, DEFAULT_POLY[m]), M + 2, N, rows[keep], cols[keep], coeffs[keep])
    w = np.bincount(cols[keep], minlength=N)
    assert set(w.tolist()) == {1, 2, 3}
    _agree(code, rng.normal(1.0, 1.8, N * m), 4)

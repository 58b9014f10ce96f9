"""Pins for the conventional Log-SP oracle (O-LS), the paper's comparison algorithm.

O-LS is pinned by its initialisation against the independent bit-product prior, by per-edge,
per-iteration agreement with the probability-domain O-SP ("the outputs of this
Log-SP algorithm is the same as those of the SP algorithm"), by exact symbol-MAP decisions on
a cycle-free code, and by end-to-end properties (noiseless frames, codeword outputs)."""
import numpy as np
import pytest

import oracle
import synth
from helpers import DEFAULT_POLY, bit_prior, enumerate_codewords


def _code(m, N, k, seed):
    M, rows, cols, coeffs = synth.make_regular_code(N, k, m, seed)
    return oracle.Code(oracle.Field(m, DEFAULT_POLY[m]), M, N, rows, cols, coeffs)


def test_ls_init_is_log_of_bit_prior():
    m, N = 4, 8
    code = _code(m, N, 4, 61)
    llr = np.random.default_rng(61).normal(0.5, 3.0, N * m)
    L0 = code.ls_init(llr)
    for v in range(N):
        np.testing.assert_allclose(np.exp(L0[v]), bit_prior(llr[v * m:(v + 1) * m]), rtol=1e-12)
    pmf = np.random.default_rng(62).random((N, 1 << m))
    np.testing.assert_allclose(code.ls_init_pmf(pmf), np.log(pmf), rtol=1e-14)


@pytest.mark.parametrize("m,N,k,seed", [(2, 16, 4, 71), (3, 12, 4, 72), (4, 12, 3, 73), (5, 8, 4, 74)])
def test_ls_equals_sp_per_edge_per_iteration(m, N, k, seed):
    code = _code(m, N, k, seed)
    rng = np.random.default_rng(seed)
    llr = rng.normal(1.2, 1.8, N * m)
    p0 = code.sp_init(llr)
    L0 = code.ls_init(llr)
    _, ecol, _ = code.edges()
    u, V = p0[ecol].copy(), L0[ecol].copy()
    for _ in range(5):
        w = code.sp_check_to_variable(u)
        W = code.ls_check_to_variable(V)
        # the log-convolution is the log of the convolution: equal up to a per-edge constant
        np.testing.assert_allclose(W - W[:, :1], np.log(w) - np.log(w[:, :1]), rtol=1e-9, atol=1e-9)
        u = code.sp_variable_to_check(p0, w, norm_mode=1)
        V = code.ls_variable_to_check(L0, W)
        np.testing.assert_allclose(V, np.log(u), rtol=1e-9, atol=1e-9)
        qv = code.sp_posterior(p0, w)
        x, mu = code.ls_decision(L0, W)
        post = np.exp(mu - mu.max(1, keepdims=True))
        post /= post.sum(1, keepdims=True)
        np.testing.assert_allclose(post, qv, rtol=1e-8, atol=1e-14)
        top2 = np.sort(qv, 1)[:, -2:]
        clear = top2[:, 1] - top2[:, 0] > 1e-9
        assert np.array_equal(x[clear], qv.argmax(1)[clear])


def test_ls_decode_is_symbol_map_on_tree():
    m, N, rows, cols = 3, 5, [0, 0, 0, 1, 1, 1], [0, 1, 2, 2, 3, 4]
    q = 1 << m
    rng = np.random.default_rng(81)
    coeffs = rng.integers(1, q, len(rows))
    code = oracle.Code(oracle.Field(m, DEFAULT_POLY[m]), 2, N, rows, cols, coeffs)
    cw = enumerate_codewords(2, N, m, DEFAULT_POLY[m], rows, cols, coeffs)
    for _ in range(4):
        llr = rng.normal(0.6, 1.5, N * m).astype(np.float32)
        pri = np.array([bit_prior(llr[v * m:(v + 1) * m].astype(np.float64)) for v in range(N)])
        wgt = np.prod([pri[v, cw[:, v]] for v in range(N)], axis=0)
        post = np.zeros((N, q))
        for v in range(N):
            np.add.at(post[v], cw[:, v], wgt)
        r = code.ls_decode_batch(llr[None], max_iters=3, early_stop=False)
        assert np.array_equal(r["hard"][0], post.argmax(1))


def test_ls_noiseless_and_codeword_outputs():
    m, N, k = 4, 24, 4
    code = _code(m, N, k, 31)
    x, _ = code.encode(synth.random_symbols(N, 16, 31))
    llr = (1 - 2.0 * synth.symbols_to_bits(x[None], m)) * 30.0
    r = code.ls_decode_batch(llr, max_iters=10)
    assert r["iters"][0] == 1 and r["ok"][0] == 1 and np.array_equal(r["hard"][0], x.astype(np.uint8))
    c = synth.CONFIGS["C1"]
    M, rows, cols, coeffs = synth.config_code("C1")
    oc = oracle.Code(oracle.Field(c["m"], c["poly"]), M, c["N"], rows, cols, coeffs)
    llr = synth.config_llr("C1", 0, 64)
    a = oc.ls_decode_batch(llr, c["max_iters"])
    assert a["ok"].mean() > 0.75  # the LF decoder (bit-wise decisions) converges on ~80% of these
    for xh in a["hard"][a["ok"] == 1]:
        assert oc.syndrome(xh)[0]
    b = oc.ls_decode_batch(llr, c["max_iters"], f32=True)
    assert ((a["hard"] == b["hard"]).all(1) & (a["iters"] == b["iters"])).mean() > 0.9

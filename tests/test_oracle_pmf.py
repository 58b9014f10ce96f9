"""Pins for the oracle's symbol-pmf input (the general INITIALIZATION).

P_v^(0) = WHT(p_v^(0)) is pinned by closed forms (a point mass, the q-ary symmetric
channel), by the factorised prior (a bit-product pmf gives the LLR form's tensor product,
PAPER.md:641), by per-edge agreement with the probability-domain SP run on the same
non-factorisable prior, and by exact symbol-MAP bit marginals on a cycle-free code."""
import numpy as np
import pytest

import oracle
import synth
from helpers import DEFAULT_POLY, bit_prior, enumerate_codewords, hadamard


def _code(m, N, k, seed):
    M, rows, cols, coeffs = synth.make_regular_code(N, k, m, seed)
    return oracle.Code(oracle.Field(m, DEFAULT_POLY[m]), M, N, rows, cols, coeffs)


def test_point_mass_and_qsc_closed_forms():
    m, N = 3, 12
    q = 1 << m
    code = _code(m, N, 4, 3)
    rng = np.random.default_rng(3)
    y = rng.integers(0, q, N)
    par = np.array([[bin(z & x).count("1") & 1 for x in range(q)] for z in range(q)])
    # point mass at y: P(z) = (-1)^{z.y}, |P| = 1
    S0, L0 = code.lf_init_pmf(np.eye(q)[y] * 3.0)  # any positive scale
    assert np.array_equal(S0, par[:, y].T.astype(np.uint8))
    assert np.abs(L0).max() < 1e-12
    # q-ary symmetric channel: P(0) = 1, P(z) = (-1)^{z.y} (1 - eps q / (q - 1)) for z != 0
    eps = 0.2
    pmf = np.full((N, q), eps / (q - 1))
    pmf[np.arange(N), y] = 1 - eps
    S0, L0 = code.lf_init_pmf(pmf)
    c = 1 - eps * q / (q - 1)
    assert np.all(S0[:, 0] == 0) and np.abs(L0[:, 0]).max() < 1e-12
    assert np.array_equal(S0[:, 1:], par[1:, y].T.astype(np.uint8))
    np.testing.assert_allclose(L0[:, 1:], np.log(c), rtol=1e-12)  # L = ln|P|


def test_factorised_pmf_equals_llr_form():
    m, N = 4, 12
    q = 1 << m
    code = _code(m, N, 3, 5)
    llr = np.random.default_rng(5).normal(0.7, 2.0, N * m)
    pmf = np.array([bit_prior(llr[v * m:(v + 1) * m]) for v in range(N)])
    S0a, L0a = code.lf_init(llr)
    S0b, L0b = code.lf_init_pmf(pmf)
    assert np.array_equal(S0a, S0b)
    np.testing.assert_allclose(L0a, L0b, rtol=1e-9, atol=1e-11)
    assert q == pmf.shape[1]


def test_factorised_pmf_decodes_like_llr():
    c = synth.CONFIGS["C1"]
    M, rows, cols, coeffs = synth.config_code("C1")
    code = oracle.Code(oracle.Field(c["m"], c["poly"]), M, c["N"], rows, cols, coeffs)
    llr = synth.config_llr("C1", 0, 32)
    m, q, N = c["m"], c["q"], c["N"]
    pmf = np.array([[bit_prior(f[v * m:(v + 1) * m].astype(np.float64)) for v in range(N)] for f in llr])
    a = code.lf_decode_batch(llr, c["max_iters"], want_soft=True)
    b = code.lf_decode_batch_pmf(pmf.astype(np.float32), c["max_iters"], want_soft=True)
    for key in ("hard", "ok", "iters"):
        assert np.array_equal(a[key], b[key]), key
    # the float32 pmf rounds the prior at ~1e-7 relative
    np.testing.assert_allclose(a["soft"], b["soft"], atol=1e-4)


@pytest.mark.parametrize("m,N,k,seed", [(3, 12, 4, 41), (2, 16, 4, 42), (5, 8, 4, 43)])
def test_lf_from_pmf_equals_sp_per_edge(m, N, k, seed):
    # PAPER.md:329-330 with a non-factorisable prior: the Log-Fourier messages are the WHT of SP's
    code = _code(m, N, k, seed)
    q = 1 << m
    rng = np.random.default_rng(seed)
    pmf = rng.random((N, q)) ** 4 + 1e-3
    p0 = pmf / pmf.sum(1, keepdims=True)
    Hd = hadamard(m)
    S0, L0 = code.lf_init_pmf(pmf)
    np.testing.assert_allclose(np.where(S0, -1, 1) * np.exp(L0), p0 @ Hd.T, rtol=1e-9, atol=1e-14)
    _, ecol, _ = code.edges()
    u, Us, Ul = p0[ecol].copy(), S0[ecol].copy(), L0[ecol].copy()
    for _ in range(5):
        w = code.sp_check_to_variable(u)
        Ws, Wl = code.lf_check_to_variable(Us, Ul)
        Wsp = w @ Hd.T
        Wsp /= Wsp[:, :1]
        np.testing.assert_allclose(np.where(Ws, -1, 1) * np.exp(Wl), Wsp, rtol=1e-9, atol=1e-9)
        u = code.sp_variable_to_check(p0, w)
        Us, Ul, ev = code.lf_variable_to_check(S0, L0, Ws, Wl)
        assert ev == 0
        np.testing.assert_allclose(np.where(Us, -1, 1) * np.exp(Ul), u @ Hd.T, rtol=1e-9, atol=1e-9)


def test_pmf_decode_exact_on_tree():
    # checks {0,1,2},{2,3,4}: after two iterations the bit marginals are the exact ones
    m, N, rows, cols = 3, 5, [0, 0, 0, 1, 1, 1], [0, 1, 2, 2, 3, 4]
    q = 1 << m
    rng = np.random.default_rng(77)
    coeffs = rng.integers(1, q, len(rows))
    code = oracle.Code(oracle.Field(m, DEFAULT_POLY[m]), 2, N, rows, cols, coeffs)
    cw = enumerate_codewords(2, N, m, DEFAULT_POLY[m], rows, cols, coeffs)
    for _ in range(3):
        pmf = (rng.random((N, q)) ** 3 + 1e-2).astype(np.float32)
        pri = pmf.astype(np.float64)
        w = np.prod([pri[v, cw[:, v]] for v in range(N)], axis=0)
        post = np.zeros((N, q))
        for v in range(N):
            np.add.at(post[v], cw[:, v], w)
        post /= post.sum(1, keepdims=True)
        r = code.lf_decode_batch_pmf(pmf[None], max_iters=4, early_stop=False, want_soft=True)
        for v in range(N):
            for i in range(m):
                mask = ((np.arange(q) >> i) & 1).astype(bool)
                d = post[v, ~mask].sum() - post[v, mask].sum()
                assert abs(r["soft"][0, v * m + i] - np.log(abs(d))) < 1e-8
                assert ((int(r["hard"][0, v]) >> i) & 1) == int(d < 0)


def test_orthogonal_channel_pmf_decodes():
    # the seeded non-binary channel used by the GPU tests: row scale, shape, and decodability
    c = synth.CONFIGS["C1"]
    M, rows, cols, coeffs = synth.config_code("C1")
    code = oracle.Code(oracle.Field(c["m"], c["poly"]), M, c["N"], rows, cols, coeffs)
    pmf = synth.config_pmf("C1", 0, 64)
    assert pmf.shape == (64, c["N"], c["q"]) and np.allclose(pmf.max(2), 1.0)
    r = code.lf_decode_batch_pmf(pmf, c["max_iters"])
    assert r["ok"].mean() > 0.8
    for x in r["hard"][r["ok"] == 1]:  # a converged frame is a codeword ...
        assert code.syndrome(x)[0]
    # ... and decoding lowers the symbol error rate of the symbol-wise MAP decisions (N = 16 is
    # short, so some frames converge to a neighbouring codeword)
    assert (r["hard"] != 0).mean() < 0.5 * (pmf.argmax(2) != 0).mean()


@pytest.mark.parametrize("m,N,k,seed,pmf_in", [(3, 12, 4, 51, False), (4, 12, 3, 52, True), (2, 16, 4, 53, True)])
def test_symbol_posterior_equals_sp_posterior(m, N, k, seed, pmf_in):
    # mu_v = IWHT-side sum of M_v is SP's posterior (Appendix lemma); map = argmax
    code = _code(m, N, k, seed)
    q = 1 << m
    rng = np.random.default_rng(seed)
    if pmf_in:
        pmf = rng.random((N, q)) ** 4 + 1e-3
        p0 = pmf / pmf.sum(1, keepdims=True)
        S0, L0 = code.lf_init_pmf(pmf)
    else:
        llr = rng.normal(1.0, 2.0, N * m)
        p0 = code.sp_init(llr)
        S0, L0 = code.lf_init(llr)
    _, ecol, _ = code.edges()
    u, Us, Ul = p0[ecol].copy(), S0[ecol].copy(), L0[ecol].copy()
    for _ in range(4):
        w = code.sp_check_to_variable(u)
        Ws, Wl = code.lf_check_to_variable(Us, Ul)
        qv = code.sp_posterior(p0, w)
        post, xmap = code.lf_symbol_posterior(S0, L0, Ws, Wl)
        np.testing.assert_allclose(post, qv, rtol=1e-8, atol=1e-12)
        top2 = np.sort(qv, 1)[:, -2:]
        clear = top2[:, 1] - top2[:, 0] > 1e-9
        assert np.array_equal(xmap[clear], qv.argmax(1)[clear])
        u = code.sp_variable_to_check(p0, w)
        Us, Ul, _ = code.lf_variable_to_check(S0, L0, Ws, Wl)


def test_symbol_posterior_exact_on_tree():
    m, N, rows, cols = 2, 7, [0, 0, 0, 1, 1, 1, 2, 2, 2], [0, 1, 2, 2, 3, 4, 4, 5, 6]
    q = 1 << m
    rng = np.random.default_rng(91)
    coeffs = rng.integers(1, q, len(rows))
    code = oracle.Code(oracle.Field(m, DEFAULT_POLY[m]), 3, N, rows, cols, coeffs)
    cw = enumerate_codewords(3, N, m, DEFAULT_POLY[m], rows, cols, coeffs)
    pmf = (rng.random((N, q)) ** 2 + 1e-2).astype(np.float32)
    pri = pmf.astype(np.float64)
    wgt = np.prod([pri[v, cw[:, v]] for v in range(N)], axis=0)
    post = np.zeros((N, q))
    for v in range(N):
        np.add.at(post[v], cw[:, v], wgt)
    post /= post.sum(1, keepdims=True)
    r = code.lf_decode_batch_pmf(pmf[None], max_iters=4, early_stop=False, want_post=True)
    np.testing.assert_allclose(r["post"][0], post, rtol=1e-9, atol=1e-13)
    assert np.array_equal(r["map"][0], post.argmax(1))

"""Pins for the oracle's decoders: O-SP and O-LF.

O-SP is pinned by exhaustive symbol-MAP on cycle-free codes;
O-LF is pinned by per-edge, per-iteration agreement with O-SP (PAPER.md:329-330,
the Appendix lemma), by exact bit marginals on the tree, and by the fast-rule
identities."""
import numpy as np
import pytest

import oracle
import synth
from helpers import DEFAULT_POLY, bit_prior, clmul_mod, enumerate_codewords, hadamard


def _brute_posteriors(M, N, m, rows, cols, coeffs, llr):
    cw = enumerate_codewords(M, N, m, DEFAULT_POLY[m], rows, cols, coeffs)
    q = 1 << m
    pri = np.array([bit_prior(llr[v * m:(v + 1) * m]) for v in range(N)])
    w = np.prod([pri[v, cw[:, v]] for v in range(N)], axis=0)
    post = np.zeros((N, q))
    for v in range(N):
        np.add.at(post[v], cw[:, v], w)
    return post / post.sum(axis=1, keepdims=True)


TREES = [
    # (m, N, rows, cols): checks {0,1,2},{2,3,4}(,{4,5,6}); leaves have column weight 1
    (3, 5, [0, 0, 0, 1, 1, 1], [0, 1, 2, 2, 3, 4]),
    (2, 7, [0, 0, 0, 1, 1, 1, 2, 2, 2], [0, 1, 2, 2, 3, 4, 4, 5, 6]),
]


@pytest.mark.parametrize("tree", TREES)
def test_sp_and_lf_exact_on_tree(tree):
    m, N, rows, cols = tree
    q = 1 << m
    rng = np.random.default_rng(5 + m)
    coeffs = rng.integers(1, q, len(rows))
    M = max(rows) + 1
    f = oracle.Field(m, DEFAULT_POLY[m])
    code = oracle.Code(f, M, N, rows, cols, coeffs)
    for trial in range(3):
        llr = rng.normal(0.8, 1.6, N * m)
        post = _brute_posteriors(M, N, m, rows, cols, coeffs, llr)
        # O-SP: after enough iterations (tree depth) the posterior is exact
        p0 = code.sp_init(llr)
        u = np.repeat(p0[np.array(code.edges()[1])][None], 1, 0)[0]
        for _ in range(4):
            w = code.sp_check_to_variable(u)
            u = code.sp_variable_to_check(p0, w)
        np.testing.assert_allclose(code.sp_posterior(p0, w), post, rtol=1e-10, atol=1e-13)
        # O-LF: fast bits and soft values equal the exact bit marginals
        res = code.lf_decode_batch(llr.astype(np.float32)[None], max_iters=4, early_stop=False, want_soft=True)
        llr32 = llr.astype(np.float32).astype(np.float64)
        post32 = _brute_posteriors(M, N, m, rows, cols, coeffs, llr32)
        for v in range(N):
            for i in range(m):
                mask = ((np.arange(q) >> i) & 1).astype(bool)
                d = post32[v, ~mask].sum() - post32[v, mask].sum()   # q_i(0) - q_i(1)
                assert abs(res["soft"][0, v * m + i] - np.log(abs(d))) < 1e-8
                assert ((int(res["hard"][0, v]) >> i) & 1) == int(d < 0)


def _sp_lf_agreement(code, llr, iters, tol=1e-9):
    q = code.q
    Hd = hadamard(code.m)
    _, ecol, _ = code.edges()
    p0 = code.sp_init(llr)
    S0, L0 = code.lf_init(llr)
    np.testing.assert_allclose(np.where(S0, -1, 1) * np.exp(L0), p0 @ Hd.T, rtol=1e-9, atol=1e-14)
    u = p0[ecol].copy()
    Us, Ul = S0[ecol].copy(), L0[ecol].copy()
    for it in range(iters):
        w = code.sp_check_to_variable(u)
        Ws, Wl = code.lf_check_to_variable(Us, Ul)
        Wsp = w @ Hd.T
        Wsp /= Wsp[:, :1]
        np.testing.assert_allclose(np.where(Ws, -1, 1) * np.exp(Wl), Wsp, rtol=tol, atol=tol)
        u = code.sp_variable_to_check(p0, w)
        Us, Ul, ev = code.lf_variable_to_check(S0, L0, Ws, Wl)
        assert ev == 0
        Usp = u @ Hd.T
        np.testing.assert_allclose(np.where(Us, -1, 1) * np.exp(Ul), Usp, rtol=tol, atol=tol)
        # decisions: fast-rule bits vs bit-MAP from the SP posterior, away from ties
        qv = code.sp_posterior(p0, w)
        x, soft, _ = code.lf_decision(S0, L0, Ws, Wl)
        for v in range(code.N):
            for i in range(code.m):
                mask = ((np.arange(q) >> i) & 1).astype(bool)
                d = qv[v, ~mask].sum() - qv[v, mask].sum()
                if abs(d) > 1e-6:
                    assert ((x[v] >> i) & 1) == int(d < 0)
                    assert abs(soft[v, i] - np.log(abs(d))) < 1e-6


@pytest.mark.parametrize("m,N,k,seed", [(3, 12, 4, 1), (4, 12, 3, 2), (2, 16, 4, 3), (6, 8, 4, 4)])
def test_lf_equals_sp_per_edge_per_iteration(m, N, k, seed):
    # PAPER.md:329-330 ("outputs the same decoding results"), Appendix lemma :674-680.
    M, rows, cols, coeffs = synth.make_regular_code(N, k, m, seed)
    code = oracle.Code(oracle.Field(m, DEFAULT_POLY[m]), M, N, rows, cols, coeffs)
    rng = np.random.default_rng(seed)
    llr = rng.normal(1.5, 1.8, N * m)
    _sp_lf_agreement(code, llr, iters=6)


def test_sp_normalisation_invariance():
    # value-at-0 normalisation leaves the decisions unchanged
    m, N, k = 3, 12, 4
    M, rows, cols, coeffs = synth.make_regular_code(N, k, m, 9)
    code = oracle.Code(oracle.Field(m, DEFAULT_POLY[m]), M, N, rows, cols, coeffs)
    llr = np.random.default_rng(9).normal(1.0, 2.0, N * m)
    p0 = code.sp_init(llr)
    ecol = code.edges()[1]
    ua, ub = p0[ecol].copy(), p0[ecol].copy()
    for _ in range(5):
        wa, wb = code.sp_check_to_variable(ua), code.sp_check_to_variable(ub)
        ua, ub = code.sp_variable_to_check(p0, wa, 0), code.sp_variable_to_check(p0, wb, 1)
        qa, qb = code.sp_posterior(p0, wa), code.sp_posterior(p0, wb)
        np.testing.assert_allclose(qa, qb, rtol=1e-9)
        assert np.array_equal(qa.argmax(1), qb.argmax(1))


def test_fast_bit_rule_marginal_identity():
    # Q(alpha^{i-1}) = q_i(0) - q_i(1) for any distribution q
    rng = np.random.default_rng(11)
    for m in (2, 3, 5):
        q = 1 << m
        for _ in range(50):
            qq = rng.random(q) ** 3
            qq /= qq.sum()
            Q = oracle.wht(qq)
            for i in range(m):
                mask = ((np.arange(q) >> i) & 1).astype(bool)
                assert abs(Q[1 << i] - (qq[~mask].sum() - qq[mask].sum())) < 1e-14


def test_fast_syndrome_counterexample_regression():
    # Reading R13: the paper's fast syndrome is not the syndrome of
    # the fast-rule bits in general.  GF(4), q_v = (0.4, 0.3, 0.3, 0): Q(1) = Q(2) = 0.4 > 0
    # so xhat_v = 0, yet Q(3) = -0.2 < 0: a check with H_cv alpha^{i-1} = 3 sees a "1".
    f = oracle.Field(2, 0x7)
    Q = oracle.wht([0.4, 0.3, 0.3, 0.0])
    assert Q[1] > 0 and Q[2] > 0 and Q[3] < 0
    hits = [(h, i) for h in range(1, 4) for i in range(2) if f.fourier_perm(h, 1 << i) == 3]
    assert hits, "some coefficient maps a unit vector to 3"


def test_fast_syndrome_equals_exact_when_confident():
    # Under top-symbol mass > 1/2 for every variable of a check the two rules agree.
    m, N, k = 3, 24, 4
    M, rows, cols, coeffs = synth.make_regular_code(N, k, m, 21)
    code = oracle.Code(oracle.Field(m, DEFAULT_POLY[m]), M, N, rows, cols, coeffs)
    rng = np.random.default_rng(21)
    checked = 0
    for trial in range(20):
        x, _ = code.encode(rng.integers(0, 8, N))
        bits = synth.symbols_to_bits(x[None], m)[0]
        llr = (1 - 2.0 * bits) * 3.0 + rng.normal(0, 2.0, N * m)
        p0 = code.sp_init(llr)
        S0, L0 = code.lf_init(llr)
        ecol = code.edges()[1]
        u, Us, Ul = p0[ecol], S0[ecol], L0[ecol]
        for _ in range(2):
            w = code.sp_check_to_variable(u)
            Ws, Wl = code.lf_check_to_variable(Us, Ul)
            u = code.sp_variable_to_check(p0, w)
            Us, Ul, _ = code.lf_variable_to_check(S0, L0, Ws, Wl)
            qv = code.sp_posterior(p0, w)
            xh, _, pb = code.lf_decision(S0, L0, Ws, Wl)
            _, s = code.syndrome(xh)
            erow, ecol2, eh = code.edges()
            for c in range(M):
                vs = ecol2[erow == c]
                if np.all(qv[vs].max(1) > 0.5):
                    assert pb[c] == s[c]
                    checked += 1
    assert checked > 100


@pytest.mark.parametrize("name", ["C1", "C3"])
def test_encoder_produces_codewords(name):
    c = synth.CONFIGS[name]
    M, rows, cols, coeffs = synth.config_code(name)
    code = oracle.Code(oracle.Field(c["m"], c["poly"]), M, c["N"], rows, cols, coeffs)
    erow, ecol, eh = code.edges()
    for t in range(3):
        x, rank = code.encode(synth.random_symbols(c["N"], c["q"], c["seed_codeword"], t))
        assert 0 < rank <= M
        # H x = 0 via carry-less products (independent of the oracle's tables)
        s = np.zeros(M, np.int64)
        for r, v, h in zip(erow, ecol, eh):
            s[r] ^= clmul_mod(int(h), int(x[v]), c["m"], c["poly"])
        assert not s.any()
        assert code.syndrome(x)[0]
        assert len(set(x.tolist())) > 1
    y = x.copy()
    y[0] ^= 1
    assert not code.syndrome(y)[0]


def test_noiseless_converges_at_first_iteration():
    # zero-noise transmission converges at l = 1 to the codeword
    m, N, k = 4, 24, 4
    M, rows, cols, coeffs = synth.make_regular_code(N, k, m, 31)
    code = oracle.Code(oracle.Field(m, DEFAULT_POLY[m]), M, N, rows, cols, coeffs)
    x, _ = code.encode(synth.random_symbols(N, 16, 31))
    llr = (1 - 2.0 * synth.symbols_to_bits(x[None], m)) * 30.0
    for mode in (oracle.EXACT, oracle.PAPER):
        r = code.lf_decode_batch(llr, max_iters=10, mode=mode)
        assert r["iters"][0] == 1 and r["ok"][0] == 1
        assert np.array_equal(r["hard"][0], x.astype(np.uint8))


def test_check_degree_two_passes_message_through():
    # k = 2, the outgoing message is the other incoming one, permuted
    m = 3
    f = oracle.Field(m, DEFAULT_POLY[m])
    code = oracle.Code(f, 1, 2, [0, 0], [0, 1], [3, 5])
    rng = np.random.default_rng(4)
    Ul = -rng.random((2, 8)) * 3
    Ul[:, 0] = 0
    Us = rng.integers(0, 2, (2, 8)).astype(np.uint8)
    Us[:, 0] = 0
    Ws, Wl = code.lf_check_to_variable(Us, Ul)
    for z in range(8):
        w = f.fourier_perm_inv(3, z)
        zz = f.fourier_perm(5, w)
        assert Wl[0, z] == Ul[1, zz] and Ws[0, z] == Us[1, zz]


def test_f32_twin_tracks_f64_on_c1():
    c = synth.CONFIGS["C1"]
    M, rows, cols, coeffs = synth.config_code("C1")
    code = oracle.Code(oracle.Field(c["m"], c["poly"]), M, c["N"], rows, cols, coeffs)
    llr = synth.config_llr("C1", 0, 64)
    a = code.lf_decode_batch(llr, c["max_iters"])
    b = code.lf_decode_batch(llr, c["max_iters"], f32=True)
    same = (a["hard"] == b["hard"]).all(1) & (a["ok"] == b["ok"]) & (a["iters"] == b["iters"])
    assert same.mean() > 0.9


try:
    from hypothesis import given, settings, strategies as st

    @settings(max_examples=25, deadline=None, derandomize=True)
    @given(m=st.integers(1, 4), k=st.sampled_from([3, 4, 6]), half_n=st.integers(3, 8), seed=st.integers(0, 10**6),
           mu=st.floats(-1.0, 2.5), sd=st.floats(0.3, 3.0))
    def test_lf_equals_sp_random_codes(m, k, half_n, seed, mu, sd):
        # PAPER.md:329-330 on randomly drawn (2,k) codes, fields and channels: O-LF's messages are the
        # WHT of O-SP's, edge by edge, for three iterations
        N = half_n * k
        M, rows, cols, coeffs = synth.make_regular_code(N, k, m, seed)
        code = oracle.Code(oracle.Field(m, DEFAULT_POLY[m]), M, N, rows, cols, coeffs)
        llr = np.random.default_rng(seed).normal(mu, sd, N * m)
        _sp_lf_agreement(code, llr, iters=3, tol=1e-8)
except ImportError:  # pragma: no cover
    pass

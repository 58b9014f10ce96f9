"""Pins for O-LF-half, the oracle of the half-precision message format (NBLDPC_MSG_F16; SURVEY 8(f)
row 4, the quantisation motivation of PAPER.md:57-71; reading R26 in DESIGN.md): O-LF with every
stored check-to-variable message rounded -- sign kept, -log2|x| rounded to IEEE binary16 -- after each
check node.  The rounding is a storage rule, not new arithmetic, so it is pinned against an independent
implementation of the format (numpy's float16 conversion, a library primitive), and the decoder is
pinned against O-LF where the rule is the identity and against the rule applied step by step."""
import numpy as np
import pytest

import oracle
import synth
from helpers import DEFAULT_POLY
from parity import config_inputs, oracle_code

LN2 = np.log(2.0)


def test_round_half_matches_ieee_binary16():
    rng = np.random.default_rng(7)
    vals = np.concatenate([
        np.exp2(rng.uniform(-27, 17, 20000)),                       # log-uniform over the whole range
        (rng.integers(1, 2047, 2000) + 0.5) * 2.0 ** -10,            # exact ties in [1, 2)
        (rng.integers(1, 2047, 2000) + 0.5) * 2.0 ** 4,              # exact ties in [2^14, 2^15)
        (rng.integers(0, 1024, 2000) + 0.5) * 2.0 ** -24,            # ties among subnormals
        np.array([65504.0, 65519.9, 65520.0, 1e6, 2.0 ** -24, 2.0 ** -25, 2.0 ** -25 * 1.0001, 0.0]),
    ])
    vals = np.concatenate([vals, -vals[:500]])
    with np.errstate(over="ignore"):
        want = vals.astype(np.float16).astype(np.float64)
    got = np.array([oracle.round_half(v) for v in vals])
    assert np.array_equal(got, want), vals[got != want][:5]


def test_round_half_toward_zero():
    """The diagnostic second rounding: the largest binary16 value not above |v| in magnitude."""
    rng = np.random.default_rng(8)
    vals = np.exp2(rng.uniform(-26, 16, 5000))
    for v in vals:
        r = oracle.round_half(v, toward_zero=True)
        assert r <= v and float(np.float16(r)) == r  # representable, not above
        up = float(np.nextafter(np.float16(r), np.float16(np.inf)))
        assert up > v or up == r  # the next binary16 value is above v
        assert oracle.round_half(-v, toward_zero=True) == -r


def test_store_half_is_the_rounding_rule_entrywise():
    """On messages the oracle's check node produces (C2 and a GF(256) code), lf_store_half writes
    ln' = -ln 2 * fp16(-ln / ln 2) with the sign kept, and leaves zeros (the floor) alone."""
    for name in ("C2", "C3"):
        c = synth.CONFIGS[name]
        code = oracle_code(name)
        _, llr, _ = config_inputs(name, 0, 1)
        S0, L0 = code.lf_init(llr[0].astype(np.float64))
        ecol = code.edges()[1]
        Ws, Wl = code.lf_check_to_variable(S0[ecol], L0[ecol])
        hs, hl = code.lf_store_half(Ws, Wl)
        zero = Wl <= oracle.FLOOR
        mag16 = (-Wl / LN2).astype(np.float16).astype(np.float64)
        want = np.where(zero, Wl, -mag16 * LN2)
        want = np.maximum(want, oracle.FLOOR)
        assert np.array_equal(hl, want)
        assert np.array_equal(hs, np.where(want <= oracle.FLOOR, 0, Ws))
        # 11 significant bits (an absolute 2^-25 ln 2 among binary16 subnormals; magnitudes are >= 0)
        bound = np.maximum(np.abs(Wl) * 2.0 ** -11, 2.0 ** -25 * LN2) + np.maximum(Wl, 0.0)
        assert (np.abs(hl - Wl)[~zero] <= bound[~zero]).all()
        assert not np.array_equal(hl, Wl)  # the rule is not the identity on real messages


def test_half_decoder_equals_lf_where_the_rule_is_the_identity():
    """Noiseless and erased channels: every message is (0, 0) or zero, which binary16 holds exactly, so
    O-LF-half and O-LF give identical decodes (hard, ok, iterations, soft)."""
    c = synth.CONFIGS["C1"]
    code = oracle_code("C1")
    _, llr, xs = config_inputs("C1", 0, 8)
    bits = synth.symbols_to_bits(xs, c["m"]).astype(np.float32)
    for x in (1e4 * (1 - 2 * bits), np.zeros_like(llr)):
        a = code.lf_decode_batch(x, 5, want_soft=True)
        b = code.lf_decode_batch(x, 5, want_soft=True, half=True)
        for k in ("hard", "ok", "iters", "soft"):
            assert np.array_equal(a[k], b[k]), k


def test_half_decoder_applies_the_rule_after_each_check_node():
    """One and two iterations of O-LF-half equal the O-LF steps with lf_store_half applied to every W:
    the soft outputs of the decode are those of the rounded state."""
    for name in ("C1", "C2"):
        c = synth.CONFIGS[name]
        code = oracle_code(name)
        _, llr, _ = config_inputs(name, 0, 2)
        ecol = code.edges()[1]
        for f in range(2):
            S0, L0 = code.lf_init(llr[f].astype(np.float64))
            Us, Ul = S0[ecol].copy(), L0[ecol].copy()
            for it in (1, 2):
                Ws, Wl = code.lf_store_half(*code.lf_check_to_variable(Us, Ul))
                x, soft, _ = code.lf_decision(S0, L0, Ws, Wl)
                Us, Ul, _ = code.lf_variable_to_check(S0, L0, Ws, Wl)
                r = code.lf_decode_batch(llr[f:f + 1], it, early_stop=False, want_soft=True, half=True)
                assert np.array_equal(r["hard"][0], x)
                assert np.array_equal(r["soft"][0], soft.ravel()), (name, f, it)


def test_half_decoder_decodes_like_lf():
    """Quality report, not a pin: on C1 the half-precision store changes few decisions."""
    code = oracle_code("C1")
    c = synth.CONFIGS["C1"]
    _, llr, _ = config_inputs("C1", 0, 64)
    a = code.lf_decode_batch(llr, c["max_iters"])
    b = code.lf_decode_batch(llr, c["max_iters"], half=True)
    assert ((a["hard"] == b["hard"]).all(1)).mean() >= 0.9

"""Shared helpers for the GPU parity tests (tests/ only; imports the oracle).

Message formats:
  GPU  : packed float32, magnitude = -log2|x| (>= 0, 200 = zero), IEEE sign bit = sign
  oracle: (sign uint8, ln|x| float64 with floor -745)
"""
from __future__ import annotations

import numpy as np

import oracle
import synth

LN2 = np.log(2.0)
ZERO_LN = -87.0  # entries at or below e^-87 are "zero" for comparisons (reading R7)


def oracle_code(name_or_cfg, M=None, rows=None, cols=None, coeffs=None):
    if isinstance(name_or_cfg, str):
        c = synth.CONFIGS[name_or_cfg]
        M, rows, cols, coeffs = synth.config_code(name_or_cfg)
    else:
        c = name_or_cfg
    return oracle.Code(oracle.Field(c["m"], c["poly"]), M, c["N"], rows, cols, coeffs)


def config_inputs(name, frame0, nframes, point=0, ebn0=None):
    """(code tuple, llr float32 [F, N*m], sent symbols [F, N]) for a BASELINE config."""
    c = synth.CONFIGS[name]
    M, rows, cols, coeffs = synth.config_code(name)
    if c["codeword"] == "random":
        ocode = oracle_code(name)
        xs = np.stack([ocode.encode(synth.random_symbols(c["N"], c["q"], c["seed_codeword"], f))[0]
                       for f in range(frame0, frame0 + nframes)])
        bits = synth.symbols_to_bits(xs, c["m"])
    else:
        xs = np.zeros((nframes, c["N"]), np.int32)
        bits = None
    llr = synth.config_llr(name, frame0, nframes, ebn0_db=ebn0, bits=bits, point=point)
    return (M, rows, cols, coeffs), llr, xs


def packed_to_oracle(p):
    """GPU packed float32 -> (sign uint8, ln float64) with the oracle's floor."""
    p = np.asarray(p, np.float32)
    mag = np.abs(p).astype(np.float64)
    s = (np.signbit(p)).astype(np.uint8)
    l = -mag * LN2
    zero = mag >= 200.0
    l[zero] = oracle.FLOOR
    s[zero] = 0
    return s, l


def oracle_to_packed(s, l):
    mag = np.minimum(-np.asarray(l, np.float64) / LN2, 200.0)
    mag = np.maximum(mag, 0.0).astype(np.float32)
    out = mag.copy()
    neg = (np.asarray(s) == 1) & (mag < 200.0)
    out[neg] = -mag[neg]
    out[neg & (mag == 0)] = np.float32(-0.0)
    return out


def message_mismatch(gs, gl, os_, ol, ln_tol=1e-3, lin_tol=1e-4):
    """Boolean mask of entries that fail the combined tolerance:
    pass if |d ln| <= ln_tol, or |d linear| <= lin_tol; a sign mismatch passes only where the
    oracle's |linear| <= lin_tol; entries that are zero on both sides pass."""
    gl = np.where(gl <= ZERO_LN, -np.inf, gl)
    ol = np.where(ol <= ZERO_LN, -np.inf, ol)
    glin = np.where(gs == 1, -1.0, 1.0) * np.exp(gl)
    olin = np.where(os_ == 1, -1.0, 1.0) * np.exp(ol)
    with np.errstate(invalid="ignore"):
        dln = np.abs(gl - ol)
    dln = np.where(np.isinf(gl) & np.isinf(ol), 0.0, dln)
    dlin = np.abs(glin - olin)
    ok_val = (dln <= ln_tol) | (dlin <= lin_tol)
    sign_ok = (gs == os_) | (np.abs(olin) <= lin_tol) | (np.isinf(gl) & np.isinf(ol))
    return ~(ok_val & sign_ok)


def soft_mismatch(g, ref, ln_tol=1e-3, lin_tol=1e-4, ln_floor=-5.0):
    """The north-star bar on posterior bit log-magnitudes soft = ln|M_v(alpha^i)/M_v(0)| (BASELINE.json
    north_star): within ``ln_tol`` in ln wherever the oracle's value is >= ln_floor,
    elsewhere within ``lin_tol`` in linear value.  Returns the boolean mask of failing entries."""
    g = np.asarray(g, np.float64)
    ref = np.asarray(ref, np.float64)
    with np.errstate(over="ignore", invalid="ignore"):
        dln = np.abs(g - ref)
        dlin = np.abs(np.exp(g) - np.exp(ref))
    return np.where(ref >= ln_floor, ~(dln <= ln_tol), ~(dlin <= lin_tol))


def stable_frames(ocode, llr, max_iters, mode=0):
    """Oracle f64 results plus the stable-frame mask (f64 and f32 twins agree; reading R20)."""
    a = ocode.lf_decode_batch(llr, max_iters, mode=mode)
    b = ocode.lf_decode_batch(llr, max_iters, mode=mode, f32=True)
    stable = (a["hard"] == b["hard"]).all(1) & (a["ok"] == b["ok"]) & (a["iters"] == b["iters"])
    return a, stable


def fail_trajectory_stable(decode, x_row, max_iters, **kw):
    """Reading R20 for a frame the oracle does not converge on (ok = 0 at max_iters): its f64 and
    f32 trajectories must also agree at max_iters - 5 and max_iters - 10 iterations before it counts
    as stable -- a chaotic non-converged frame can coincide at the last iteration by chance (C5 at
    4.5 dB: frame 1999 agrees at 50 and 49 iterations, differs by 2 symbols at 30, 40 and 45).
    ``decode`` is the oracle's batch decode (lf_decode_batch, lf_decode_batch_pmf or ls_decode_batch)."""
    kw = {k: v for k, v in kw.items() if k != "early_stop"}
    for it in (max_iters - 5, max_iters - 10):
        if it < 1:
            continue
        a = decode(x_row[None], it, early_stop=False, **kw)
        b = decode(x_row[None], it, early_stop=False, f32=True, **kw)
        if not np.array_equal(a["hard"][0], b["hard"][0]):
            return False
    return True



def assert_stable_parity(decode, x, out, ref, max_iters, max_unstable_frac=0.1, what="", also=None, **kw):
    """The stable-frame protocol (readings R20, R26): every frame whose oracle outcome is
    robust must be bit-identical (hard symbols, syndrome flag, iterations) on the GPU; differing frames
    must be unstable ones and at most ``max_unstable_frac`` of the sample.
    A frame is stable when the oracle's fp64 run (``ref``) agrees with its fp32 twin and with every
    variant in ``also`` (extra keyword sets for ``decode``, e.g. O-LF without the half store for the F16
    path) -- at the stopping iteration, and for a converged frame also one iteration before it (a frame
    whose last symbol settles at the last moment converges one iteration earlier or later under any
    rounding difference); a frame the oracle does not converge on must also agree 5 and 10 iterations
    before the end (fail_trajectory_stable).
    ``decode`` is the oracle's batch decode (lf_decode_batch / lf_decode_batch_pmf / ls_decode_batch),
    ``x`` its input rows, ``out`` numpy GPU outputs {hard, ok, iters}, ``ref`` the oracle's (fp64) result.
    Returns the number of (unstable) differing frames."""
    hard, ok, it = out["hard"], out["ok"], out["iters"]
    same = (hard == ref["hard"]).all(1) & (ok == ref["ok"]) & (it == ref["iters"])
    bad = np.where(~same)[0]
    variants = [dict(f32=True)] + [dict(v) for v in (also or [])]
    base_kw = {k: v for k, v in kw.items() if k != "early_stop"}

    def agree(a, b, n, m):
        return np.array_equal(a["hard"][n], b["hard"][m]) and a["ok"][n] == b["ok"][m] and a["iters"][n] == b["iters"][m]

    if bad.size:
        runs = [decode(x[bad], max_iters, **{**kw, **v}) for v in variants]
        for n, b in enumerate(bad):
            stable = all(agree(r, ref, n, b) for r in runs)
            if stable and ref["ok"][b] == 1 and ref["iters"][b] > 1:
                before = ref["iters"][b] - 1
                r0 = decode(x[b][None], before, early_stop=False, **base_kw)
                stable = all(np.array_equal(decode(x[b][None], before, early_stop=False, **{**base_kw, **v})["hard"][0],
                                            r0["hard"][0]) for v in variants)
            if stable and ref["ok"][b] == 0:
                stable = fail_trajectory_stable(decode, x[b], max_iters, **kw) and all(
                    fail_trajectory_stable(decode, x[b], max_iters, **{**kw, **v}) for v in variants[1:])
            assert not stable, (f"{what}: stable frame {b} differs: gpu iters {it[b]} ok {ok[b]} vs oracle "
                                f"{ref['iters'][b]} {ref['ok'][b]}, {int((hard[b] != ref['hard'][b]).sum())} symbols")
    assert bad.size <= max(1, int(max_unstable_frac * len(hard))), (what, bad.size, len(hard))
    return int(bad.size)

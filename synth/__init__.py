"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no GF(2^m) field operations,
no transforms, no message updates): it only draws random graphs, random symbols
and BPSK/AWGN channel LLRs from seeded generators, so that both sides of every
parity test receive the same bytes.  Codewords for the random-codeword configs
(C1, C3) are produced by the oracle's encoder from the symbols drawn here
(tests only); the benchmark workload (C2) uses the all-zero codeword.

Input recipe (the paper runs no experiments, so there is
no dataset to stand in for):
  * H: (2,k)-regular socket permutation with local swap repair of double edges,
    nonzero entries uniform in GF(2^m)* (SURVEY.md finding 8).
  * channel: BPSK 0 -> +1 over AWGN, sigma^2 = 1 / (2 R Eb/N0) with the design
    rate R = 1 - 2/k, LLR = 2 y / sigma^2.
  * noise for frame f is drawn in 256-frame chunks from Philox keyed by
    (seed, chunk), so a frame's LLRs do not depend on batching or sharding.
"""

from __future__ import annotations

import numpy as np

CHUNK = 256

# BASELINE.json configs[0..4]; seeds are the SURVEY.md 8(d) proposal.
CONFIGS = {
    "C1": dict(m=2, poly=0x7, k=4, N=16, frames=64, ebn0=[2.0], max_iters=20, codeword="random"),
    "C2": dict(m=6, poly=0x43, k=4, N=1024, frames=4096, ebn0=[1.0], max_iters=50, codeword="zero"),
    "C3": dict(m=8, poly=0x11D, k=8, N=512, frames=8192, ebn0=[2.5], max_iters=30, codeword="random"),
    "C4": dict(m=8, poly=0x11D, k=16, N=2048, frames=16384, ebn0=[3.5], max_iters=30, codeword="zero"),
    "C5": dict(m=4, poly=0x13, k=32, N=4096, frames=65536, ebn0=[3.0, 3.5, 4.0, 4.5, 5.0], max_iters=50,
               codeword="zero"),
    # not in BASELINE.json: the column-weight-3 workload of the SURVEY 8(f) row 3 measurements
    "J3": dict(m=6, poly=0x43, k=6, N=1024, frames=4096, ebn0=[2.0], max_iters=50, codeword="zero", j=3),
}
for _i, (_name, _c) in enumerate(CONFIGS.items()):
    _c["name"] = _name
    _c["index"] = _i
    _c["q"] = 1 << _c["m"]
    _c.setdefault("j", 2)
    _c["M"] = _c["j"] * _c["N"] // _c["k"]
    _c["rate"] = 1.0 - _c["j"] / _c["k"]
    _c["seed_graph"] = 1000 + _i
    _c["seed_codeword"] = 2000 + _i
    _c["seed_noise"] = 3000 + _i


def make_regular_code(N: int, k: int, m: int, seed: int, j: int = 2):
    """Random (j,k)-regular H over GF(2^m) as canonical (rows, cols, coeffs), sorted by (row, col).

    Socket permutation, then local swap repair of repeated (row, col) pairs:
    a conflicting edge swaps its variable endpoint with a random other edge when
    the swap creates no new conflict.  Coefficients uniform in 1..2^m-1.
    """
    if (j * N) % k:
        raise ValueError("j*N must be divisible by k")
    M = j * N // k
    rng = np.random.Generator(np.random.PCG64(seed))
    check_of = np.repeat(np.arange(M, dtype=np.int64), k)          # socket -> check
    var_of = np.repeat(np.arange(N, dtype=np.int64), j)[rng.permutation(j * N)]
    E = j * N
    # adjacency multiset per check
    from collections import Counter

    cnt = [Counter() for _ in range(M)]
    for e in range(E):
        cnt[check_of[e]][var_of[e]] += 1

    def conflicts():
        return [e for e in range(E) if cnt[check_of[e]][var_of[e]] > 1]

    bad = conflicts()
    guard = 0
    while bad:
        guard += 1
        if guard > 1000:
            raise RuntimeError("swap repair did not converge")
        for e in bad:
            c, v = check_of[e], var_of[e]
            if cnt[c][v] <= 1:
                continue
            for _ in range(10000):
                o = int(rng.integers(E))
                co, vo = check_of[o], var_of[o]
                if co == c or vo == v:
                    continue
                if cnt[c][vo] > 0 or cnt[co][v] > 0:
                    continue
                cnt[c][v] -= 1
                cnt[co][vo] -= 1
                cnt[c][vo] += 1
                cnt[co][v] += 1
                var_of[e], var_of[o] = vo, v
                break
        bad = conflicts()
    coeffs = rng.integers(1, 1 << m, size=E)
    order = np.lexsort((var_of, check_of))
    rows = check_of[order].astype(np.int32)
    cols = var_of[order].astype(np.int32)
    return M, rows, cols, coeffs.astype(np.int32)


def config_code(name: str):
    c = CONFIGS[name]
    return make_regular_code(c["N"], c["k"], c["m"], c["seed_graph"], j=c["j"])


def random_symbols(n: int, q: int, seed: int, stream: int = 0) -> np.ndarray:
    """n symbols uniform in 0..q-1 (the encoder's free-symbol draws)."""
    rng = np.random.Generator(np.random.Philox(key=[seed, stream]))
    return rng.integers(0, q, size=n).astype(np.int32)


def symbols_to_bits(x: np.ndarray, m: int) -> np.ndarray:
    """[F][N] symbols -> [F][N*m] bits, bit i of symbol v at v*m+i."""
    x = np.asarray(x)
    sh = np.arange(m)
    b = (x[..., None] >> sh) & 1
    return b.reshape(*x.shape[:-1], x.shape[-1] * m).astype(np.uint8)


def sigma2_for(ebn0_db: float, rate: float) -> float:
    """sigma^2 = 1 / (2 R Eb/N0) for unit-energy BPSK."""
    return 1.0 / (2.0 * rate * 10.0 ** (ebn0_db / 10.0))


def awgn_llr(nbits: int, frame0: int, nframes: int, sigma2: float, seed: int, bits=None) -> np.ndarray:
    """float32 LLRs [nframes][nbits] for frames frame0 .. frame0+nframes-1.

    y = (1 - 2b) + sigma n, LLR = ln P(b=0|y)/P(b=1|y) = 2y/sigma^2.  ``bits`` is
    None (all-zero codeword) or a uint8 array [nframes][nbits] of the sent bits.
    Noise for chunk c (frames c*256 .. c*256+255) comes from Philox(key=(seed, c)).
    """
    sigma = np.sqrt(sigma2)
    out = np.empty((nframes, nbits), np.float32)
    f = frame0
    end = frame0 + nframes
    while f < end:
        c = f // CHUNK
        lo, hi = f - c * CHUNK, min(CHUNK, end - c * CHUNK)
        rng = np.random.Generator(np.random.Philox(key=[seed, c]))
        noise = rng.standard_normal((CHUNK, nbits), dtype=np.float64)[lo:hi]
        y = 1.0 + sigma * noise
        if bits is not None:
            b = np.asarray(bits[f - frame0: f - frame0 + (hi - lo)], np.float64)
            y = (1.0 - 2.0 * b) + sigma * noise
        out[f - frame0: f - frame0 + (hi - lo)] = (2.0 / sigma2) * y
        f += hi - lo
    return out


def config_llr(name: str, frame0: int, nframes: int, ebn0_db: float | None = None, bits=None, point: int = 0):
    """LLRs for config ``name`` (all-zero codeword unless ``bits`` given)."""
    c = CONFIGS[name]
    eb = c["ebn0"][point] if ebn0_db is None else ebn0_db
    s2 = sigma2_for(eb, c["rate"])
    return awgn_llr(c["N"] * c["m"], frame0, nframes, s2, c["seed_noise"] + 100 * point, bits=bits)


def orthogonal_pmf(N: int, m: int, frame0: int, nframes: int, sigma2: float, seed: int, symbols=None) -> np.ndarray:
    """float32 symbol pmfs [nframes][N][q] of q-ary orthogonal signalling over AWGN.

    A non-binary channel whose pmf does not factor over the bits (the general input of
    PAPER.md:465-473): symbol x is sent as the x-th of q orthogonal unit-energy-per-bit
    pulses, amplitude A = sqrt(m); the receiver sees r_y = A [y = x] + sigma n_y, so
    Pr(X = y | r) is proportional to exp(A r_y / sigma^2).  Rows are scaled by their
    maximum (largest entry 1).  ``symbols`` is None (all-zero codeword) or [nframes][N].
    Noise is drawn per 256-frame chunk from Philox(key=(seed, chunk)) as in awgn_llr.
    """
    q = 1 << m
    A = np.sqrt(m)
    out = np.empty((nframes, N, q), np.float32)
    f = frame0
    end = frame0 + nframes
    while f < end:
        c = f // CHUNK
        lo, hi = f - c * CHUNK, min(CHUNK, end - c * CHUNK)
        n = hi - lo
        rng = np.random.Generator(np.random.Philox(key=[seed, c]))
        noise = rng.standard_normal((CHUNK, N, q), dtype=np.float32)[lo:hi].astype(np.float64)
        r = np.sqrt(sigma2) * noise
        x = np.zeros((n, N), np.int64) if symbols is None else np.asarray(symbols[f - frame0: f - frame0 + n], np.int64)
        np.put_along_axis(r, x[..., None], np.take_along_axis(r, x[..., None], 2) + A, 2)
        ll = (A / sigma2) * r
        ll -= ll.max(axis=2, keepdims=True)
        out[f - frame0: f - frame0 + n] = np.exp(ll)
        f += n
    return out


def config_pmf(name: str, frame0: int, nframes: int, ebn0_db: float | None = None, symbols=None, point: int = 0):
    """Orthogonal-signalling pmfs for config ``name`` (same Eb/N0 points as config_llr)."""
    c = CONFIGS[name]
    eb = c["ebn0"][point] if ebn0_db is None else ebn0_db
    s2 = sigma2_for(eb, c["rate"])
    return orthogonal_pmf(c["N"], c["m"], frame0, nframes, s2, c["seed_noise"] + 7000 + 100 * point, symbols)


"""CPU oracle for arXiv:1008.4370 (Log-Fourier SP decoding of non-binary LDPC codes).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_1008_4370_b200``) never imports it, and the
two share no code: this package wraps ``oracle/oracle.c`` (plain C, fp64, built
with gcc) through ctypes.  Every C function cites the PAPER.md passage it
follows; see DESIGN.md section 3 for the readings of the paper it adopts and
section 4 for what pins each function.

Pins ("parity pinned" unless noted; tests live in tests/test_oracle_*.py):
  field tables            paper GF(8) listing, carry-less products
  Fourier permutation     Appendix A lemma, all h, m = 2..8
  WHT / convolution       scipy Hadamard matrix, convolution theorem, SPEC values
  Gamma / boxplus         homomorphism, convolution theorem
  LF init                 closed form prod tanh(L/2) (Gallager f)
  SP decoder              exhaustive MAP on a cycle-free code
  LF decoder              SP <-> LF agreement per edge per iteration
  fast bit rule           brute-force marginals
  fast syndrome           exact syndrome when top mass > 1/2; counterexample
  encoder                 H x = 0 via the companion-matrix route
  floors / neutral message / sgn(0) conventions: parity unpinned (conventions)
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = [os.path.join(_HERE, "oracle.c"), os.path.join(_HERE, "lf_body.inc"), os.path.join(_HERE, "logsp_body.inc")]
_SO = os.path.join(_HERE, "liboracle.so")
_LOCK = threading.Lock()
_LIB = None

FLOOR = -745.0  # ln of "zero" (reading R7)
EXACT = 0
PAPER = 1


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so with gcc (-O2, OpenMP)."""
    newest = max(os.path.getmtime(s) for s in _SRC)
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        tmp = _SO + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", tmp, _SRC[0], "-lm"]
        subprocess.check_call(cmd, cwd=_HERE)
        os.replace(tmp, _SO)
    return _SO


def _lib():
    global _LIB
    with _LOCK:
        if _LIB is None:
            build()
            L = ctypes.CDLL(_SO)
            vp, i32, u32, dp = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint, ctypes.c_void_p
            sig = {
                "or_field_new": (vp, [i32, u32]),
                "or_field_free": (None, [vp]),
                "or_field_q": (i32, [vp]),
                "or_gf_mul": (i32, [vp, i32, i32]),
                "or_gf_inv": (i32, [vp, i32]),
                "or_field_exp": (i32, [vp, i32]),
                "or_field_log": (i32, [vp, i32]),
                "or_fourier_perm": (i32, [vp, i32, i32]),
                "or_fourier_perm_inv": (i32, [vp, i32, i32]),
                "or_companion_pow_T": (None, [vp, i32, dp]),
                "or_apply_binary_matrix": (i32, [i32, dp, i32]),
                "or_dot_parity": (i32, [i32, i32]),
                "or_wht": (None, [i32, dp, dp]),
                "or_iwht": (None, [i32, dp, dp]),
                "or_convolve": (None, [i32, dp, dp, dp]),
                "or_boxplus": (None, [i32, dp, dp, dp, dp, dp, dp]),
                "or_gamma_inv": (ctypes.c_double, [i32, ctypes.c_double]),
                "or_channel_prior": (None, [i32, dp, dp]),
                "or_round_half": (ctypes.c_double, [ctypes.c_double]),
                "or_round_half_mode": (ctypes.c_double, [ctypes.c_double, i32]),
                "or_code_new": (vp, [vp, i32, i32, i32, dp, dp, dp]),
                "or_code_free": (None, [vp]),
                "or_code_E": (i32, [vp]),
                "or_code_edges": (None, [vp, dp, dp, dp]),
                "or_code_syndrome": (i32, [vp, dp, dp]),
                "or_code_encode": (i32, [vp, dp, dp]),
                "or_sp_init": (None, [vp, dp, dp]),
                "or_sp_check_to_variable": (None, [vp, dp, dp]),
                "or_sp_variable_to_check": (None, [vp, dp, dp, dp, i32]),
                "or_sp_posterior": (None, [vp, dp, dp, dp]),
            }
            for sfx in ("", "_f32"):
                sig["or_lf_init" + sfx] = (None, [vp, dp, dp, dp])
                sig["or_lf_check_to_variable" + sfx] = (None, [vp, dp, dp, dp, dp])
                sig["or_lf_variable_to_check" + sfx] = (None, [vp, dp, dp, dp, dp, dp, dp, dp])
                sig["or_lf_decision" + sfx] = (None, [vp, dp, dp, dp, dp, dp, dp, dp])
                sig["or_lf_decode" + sfx] = (None, [vp, dp, i32, i32, i32, dp, dp, dp, dp, dp])
                sig["or_lf_decode_batch" + sfx] = (None, [vp, dp, i32, i32, i32, i32, dp, dp, dp, dp, dp, i32])
                sig["or_lf_decode_batch_ex" + sfx] = (None, [vp, dp, i32, i32, i32, i32, i32, dp, dp, dp, dp, dp, dp,
                                                               dp, i32, i32])
                sig["or_lf_store_half" + sfx] = (None, [ctypes.c_size_t, dp, dp])
                sig["or_lf_symbol_posterior" + sfx] = (None, [vp, dp, dp, dp, dp, dp, dp])
                sig["or_lf_init_pmf" + sfx] = (None, [vp, dp, dp, dp])
                sig["or_ls_init" + sfx] = (None, [vp, dp, dp])
                sig["or_ls_init_pmf" + sfx] = (None, [vp, dp, dp])
                sig["or_ls_check_to_variable" + sfx] = (None, [vp, dp, dp])
                sig["or_ls_variable_to_check" + sfx] = (None, [vp, dp, dp, dp])
                sig["or_ls_decision" + sfx] = (None, [vp, dp, dp, dp, dp])
                sig["or_ls_decode_batch" + sfx] = (None, [vp, dp, i32, i32, i32, i32, dp, dp, dp, i32])
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _LIB = L
    return _LIB


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _u8(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint8)


# ---------------------------------------------------------------- field
class Field:
    """GF(2^m) with primitive polynomial ``poly`` (full mask incl. x^m)."""

    def __init__(self, m: int, poly: int):
        self._L = _lib()
        self.m, self.q, self.poly = m, 1 << m, poly
        self._h = self._L.or_field_new(m, poly)
        if not self._h:
            raise ValueError(f"polynomial {poly:#x} is not primitive of degree {m}")

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.or_field_free(self._h)
            self._h = None

    def mul(self, a: int, b: int) -> int:
        return self._L.or_gf_mul(self._h, int(a), int(b))

    def inv(self, a: int) -> int:
        return self._L.or_gf_inv(self._h, int(a))

    def exp(self, i: int) -> int:
        return self._L.or_field_exp(self._h, int(i))

    def log(self, x: int) -> int:
        return self._L.or_field_log(self._h, int(x))

    def fourier_perm(self, h: int, z: int) -> int:
        """z -> H_cv z with H_cv = (A^i)^T, h = alpha^i."""
        return self._L.or_fourier_perm(self._h, int(h), int(z))

    def fourier_perm_inv(self, h: int, z: int) -> int:
        return self._L.or_fourier_perm_inv(self._h, int(h), int(z))

    def perm_table(self) -> np.ndarray:
        t = np.zeros((self.q, self.q), np.int32)
        for h in range(1, self.q):
            for z in range(self.q):
                t[h, z] = self.fourier_perm(h, z)
        return t

    def companion_pow_T(self, i: int) -> np.ndarray:
        out = np.zeros(self.m * self.m, np.uint8)
        self._L.or_companion_pow_T(self._h, int(i), _p(out))
        return out.reshape(self.m, self.m)

    def apply_binary_matrix(self, mat: np.ndarray, z: int) -> int:
        mm = _u8(mat).reshape(-1)
        return self._L.or_apply_binary_matrix(self.m, _p(mm), int(z))


def dot_parity(z: int, x: int) -> int:
    return _lib().or_dot_parity(int(z), int(x))


def wht(p) -> np.ndarray:
    p = _f64(p)
    m = int(np.log2(p.size))
    out = np.zeros_like(p)
    _lib().or_wht(m, _p(p), _p(out))
    return out


def iwht(P) -> np.ndarray:
    P = _f64(P)
    m = int(np.log2(P.size))
    out = np.zeros_like(P)
    _lib().or_iwht(m, _p(P), _p(out))
    return out


def convolve(a, b) -> np.ndarray:
    a, b = _f64(a), _f64(b)
    m = int(np.log2(a.size))
    out = np.zeros_like(a)
    _lib().or_convolve(m, _p(a), _p(b), _p(out))
    return out


def gamma(x):
    """Gamma(x) = (sgn, ln|x|) elementwise; sgn(0)=0, ln 0 = FLOOR."""
    x = _f64(x)
    s = (x < 0).astype(np.uint8)
    with np.errstate(divide="ignore"):
        l = np.where(x == 0, FLOOR, np.maximum(np.log(np.abs(x)), FLOOR))
    return s, l


def gamma_inv(s, l) -> np.ndarray:
    L = _lib()
    s = np.asarray(s).reshape(-1)
    l = np.asarray(l, np.float64).reshape(-1)
    return np.array([L.or_gamma_inv(int(a), float(b)) for a, b in zip(s, l)])


def boxplus(s1, l1, s2, l2):
    s1, s2 = _i32(s1), _i32(s2)
    l1, l2 = _f64(l1), _f64(l2)
    m = int(np.log2(l1.size))
    so = np.zeros(l1.size, np.int32)
    lo = np.zeros(l1.size, np.float64)
    _lib().or_boxplus(m, _p(s1), _p(l1), _p(s2), _p(l2), _p(so), _p(lo))
    return so, lo


def round_half(v: float, toward_zero: bool = False) -> float:
    """IEEE binary16 rounding (the oracle's own, written from the format's definition): to nearest
    (ties to even), or toward zero."""
    return float(_lib().or_round_half_mode(float(v), 2 if toward_zero else 1))


def channel_prior(llr) -> np.ndarray:
    llr = _f64(llr)
    out = np.zeros(1 << llr.size)
    _lib().or_channel_prior(llr.size, _p(llr), _p(out))
    return out


# ---------------------------------------------------------------- code
class Code:
    """Tanner graph of H; edges in canonical (row, col) order."""

    def __init__(self, field: Field, M: int, N: int, rows, cols, coeffs):
        self._L = _lib()
        self.field, self.M, self.N = field, M, N
        self.m, self.q = field.m, field.q
        r, c, h = _i32(rows), _i32(cols), _i32(coeffs)
        self._h = self._L.or_code_new(field._h, M, N, r.size, _p(r), _p(c), _p(h))
        if not self._h:
            raise ValueError("invalid parity-check matrix")
        self.E = self._L.or_code_E(self._h)

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.or_code_free(self._h)
            self._h = None

    def edges(self):
        r = np.zeros(self.E, np.int32)
        c = np.zeros(self.E, np.int32)
        h = np.zeros(self.E, np.int32)
        self._L.or_code_edges(self._h, _p(r), _p(c), _p(h))
        return r, c, h

    def syndrome(self, x):
        x = _i32(x)
        s = np.zeros(self.M, np.int32)
        ok = self._L.or_code_syndrome(self._h, _p(x), _p(s))
        return bool(ok), s

    def encode(self, draws):
        """Gaussian-elimination encoder: free symbols from ``draws``; returns (x, rank)."""
        d = _i32(draws)
        x = np.zeros(self.N, np.int32)
        rank = self._L.or_code_encode(self._h, _p(d), _p(x))
        return x, rank

    # ---- SP (probability domain) steps
    def sp_init(self, llr):
        llr = _f64(llr)
        p0 = np.zeros((self.N, self.q))
        self._L.or_sp_init(self._h, _p(llr), _p(p0))
        return p0

    def sp_check_to_variable(self, u):
        u = _f64(u)
        w = np.zeros((self.E, self.q))
        self._L.or_sp_check_to_variable(self._h, _p(u), _p(w))
        return w

    def sp_variable_to_check(self, p0, w, norm_mode: int = 0):
        p0, w = _f64(p0), _f64(w)
        u = np.zeros((self.E, self.q))
        self._L.or_sp_variable_to_check(self._h, _p(p0), _p(w), _p(u), norm_mode)
        return u

    def sp_posterior(self, p0, w):
        p0, w = _f64(p0), _f64(w)
        qv = np.zeros((self.N, self.q))
        self._L.or_sp_posterior(self._h, _p(p0), _p(w), _p(qv))
        return qv

    # ---- Log-Fourier steps (double, or float32 twin with f32=True)
    def _real(self, f32):
        return (np.float32, "_f32") if f32 else (np.float64, "")

    def lf_init(self, llr, f32=False):
        dt, sfx = self._real(f32)
        llr = _f64(llr)
        S0 = np.zeros((self.N, self.q), np.uint8)
        L0 = np.zeros((self.N, self.q), dt)
        getattr(self._L, "or_lf_init" + sfx)(self._h, _p(llr), _p(S0), _p(L0))
        return S0, L0

    def lf_init_pmf(self, pmf, f32=False):
        """Lambda^(0) from a symbol-level channel pmf [N][q]."""
        dt, sfx = self._real(f32)
        pmf = _f64(pmf)
        S0 = np.zeros((self.N, self.q), np.uint8)
        L0 = np.zeros((self.N, self.q), dt)
        getattr(self._L, "or_lf_init_pmf" + sfx)(self._h, _p(pmf), _p(S0), _p(L0))
        return S0, L0

    def lf_check_to_variable(self, Us, Ul, f32=False):
        dt, sfx = self._real(f32)
        Us, Ul = _u8(Us), np.ascontiguousarray(Ul, dt)
        Ws = np.zeros((self.E, self.q), np.uint8)
        Wl = np.zeros((self.E, self.q), dt)
        getattr(self._L, "or_lf_check_to_variable" + sfx)(self._h, _p(Us), _p(Ul), _p(Ws), _p(Wl))
        return Ws, Wl

    def lf_variable_to_check(self, S0, L0, Ws, Wl, f32=False):
        dt, sfx = self._real(f32)
        S0, Ws = _u8(S0), _u8(Ws)
        L0, Wl = np.ascontiguousarray(L0, dt), np.ascontiguousarray(Wl, dt)
        Us = np.zeros((self.E, self.q), np.uint8)
        Ul = np.zeros((self.E, self.q), dt)
        ev = ctypes.c_int(0)
        getattr(self._L, "or_lf_variable_to_check" + sfx)(
            self._h, _p(S0), _p(L0), _p(Ws), _p(Wl), _p(Us), _p(Ul), ctypes.cast(ctypes.pointer(ev), ctypes.c_void_p)
        )
        return Us, Ul, ev.value

    def lf_decision(self, S0, L0, Ws, Wl, f32=False):
        dt, sfx = self._real(f32)
        S0, Ws = _u8(S0), _u8(Ws)
        L0, Wl = np.ascontiguousarray(L0, dt), np.ascontiguousarray(Wl, dt)
        x = np.zeros(self.N, np.int32)
        soft = np.zeros((self.N, self.m), dt)
        pb = np.zeros(self.M, np.int32)
        getattr(self._L, "or_lf_decision" + sfx)(self._h, _p(S0), _p(L0), _p(Ws), _p(Wl), _p(x), _p(soft), _p(pb))
        return x, soft, pb

    def lf_symbol_posterior(self, S0, L0, Ws, Wl, f32=False):
        """Symbol posterior mu_v / sum mu_v [N][q] and symbol-MAP decision [N]."""
        dt, sfx = self._real(f32)
        S0, Ws = _u8(S0), _u8(Ws)
        L0, Wl = np.ascontiguousarray(L0, dt), np.ascontiguousarray(Wl, dt)
        post = np.zeros((self.N, self.q), dt)
        xmap = np.zeros(self.N, np.int32)
        getattr(self._L, "or_lf_symbol_posterior" + sfx)(self._h, _p(S0), _p(L0), _p(Ws), _p(Wl), _p(post), _p(xmap))
        return post, xmap

    def _decode_batch(self, inp, is_pmf, max_iters, mode, early_stop, want_soft, want_post, nthreads, f32, half=False):
        dt, sfx = self._real(f32)
        row = self.N * (self.q if is_pmf else self.m)
        inp = np.ascontiguousarray(inp, np.float32).reshape(-1, row)
        F = inp.shape[0]
        x = np.zeros((F, self.N), np.int32)
        ok = np.zeros(F, np.int32)
        it = np.zeros(F, np.int32)
        ev = np.zeros(F, np.int32)
        soft = np.zeros((F, self.N * self.m), dt) if want_soft else None
        post = np.zeros((F, self.N, self.q), dt) if want_post else None
        xmap = np.zeros((F, self.N), np.int32) if want_post else None
        nt = nthreads or os.cpu_count() or 1
        opt = lambda a: _p(a) if a is not None else None  # noqa: E731
        getattr(self._L, "or_lf_decode_batch_ex" + sfx)(
            self._h, _p(inp), int(bool(is_pmf)), F, int(max_iters), int(mode), int(bool(early_stop)), _p(x), _p(ok),
            _p(it), opt(soft), _p(ev), opt(post), opt(xmap), (2 if half == "rz" else int(bool(half))), int(nt),
        )
        out = {"hard": x.astype(np.uint8), "ok": ok.astype(np.uint8), "iters": it, "events": ev}
        if soft is not None:
            out["soft"] = soft
        if want_post:
            out["post"] = post
            out["map"] = xmap.astype(np.uint8)
        return out

    # ---- conventional Log-SP, double or the float32 twin
    def ls_init(self, llr, f32=False):
        dt, sfx = self._real(f32)
        L0 = np.zeros((self.N, self.q), dt)
        getattr(self._L, "or_ls_init" + sfx)(self._h, _p(_f64(llr)), _p(L0))
        return L0

    def ls_init_pmf(self, pmf, f32=False):
        dt, sfx = self._real(f32)
        L0 = np.zeros((self.N, self.q), dt)
        getattr(self._L, "or_ls_init_pmf" + sfx)(self._h, _p(_f64(pmf)), _p(L0))
        return L0

    def ls_check_to_variable(self, V, f32=False):
        dt, sfx = self._real(f32)
        V = np.ascontiguousarray(V, dt)
        W = np.zeros((self.E, self.q), dt)
        getattr(self._L, "or_ls_check_to_variable" + sfx)(self._h, _p(V), _p(W))
        return W

    def ls_variable_to_check(self, L0, W, f32=False):
        dt, sfx = self._real(f32)
        L0, W = np.ascontiguousarray(L0, dt), np.ascontiguousarray(W, dt)
        V = np.zeros((self.E, self.q), dt)
        getattr(self._L, "or_ls_variable_to_check" + sfx)(self._h, _p(L0), _p(W), _p(V))
        return V

    def ls_decision(self, L0, W, f32=False):
        dt, sfx = self._real(f32)
        L0, W = np.ascontiguousarray(L0, dt), np.ascontiguousarray(W, dt)
        x = np.zeros(self.N, np.int32)
        mu = np.zeros((self.N, self.q), dt)
        getattr(self._L, "or_ls_decision" + sfx)(self._h, _p(L0), _p(W), _p(x), _p(mu))
        return x, mu

    def ls_decode_batch(self, inp, max_iters: int, early_stop: bool = True, pmf: bool = False,
                        nthreads: int | None = None, f32: bool = False):
        """Conventional Log-SP decode of F frames (LLRs [F][N*m] or pmfs [F][N][q]); symbol-MAP
        decisions, exact-syndrome stop."""
        _, sfx = self._real(f32)
        row = self.N * (self.q if pmf else self.m)
        inp = np.ascontiguousarray(inp, np.float32).reshape(-1, row)
        F = inp.shape[0]
        x = np.zeros((F, self.N), np.int32)
        ok = np.zeros(F, np.int32)
        it = np.zeros(F, np.int32)
        nt = nthreads or os.cpu_count() or 1
        getattr(self._L, "or_ls_decode_batch" + sfx)(self._h, _p(inp), int(bool(pmf)), F, int(max_iters),
                                                     int(bool(early_stop)), _p(x), _p(ok), _p(it), int(nt))
        return {"hard": x.astype(np.uint8), "ok": ok.astype(np.uint8), "iters": it}

    def lf_decode_batch(self, llr, max_iters: int, mode: int = EXACT, early_stop: bool = True,
                        want_soft: bool = False, nthreads: int | None = None, f32: bool = False,
                        want_post: bool = False, half: bool = False):
        """Decode F frames (llr float32 [F][N*m]); returns dict of numpy arrays (hard, ok, iters,
        events; soft [F][N*m]; post [F][N][q] and map [F][N] at the stopping iteration).
        half=True: O-LF-half, the stored messages rounded to the half-precision format after every
        check node (lf_store_half; reading R26); half="rz": the same store rounding toward zero (a
        diagnostic second rounding of the format, for the stable-frame classification of the F16 path)."""
        return self._decode_batch(llr, False, max_iters, mode, early_stop, want_soft, want_post, nthreads, f32, half)

    def lf_store_half(self, Ws, Wl, f32=False):
        """The O-LF-half storage rule applied to a message array (sign, ln): -log2|x| rounded to IEEE
        binary16.  Returns new arrays."""
        dt, sfx = self._real(f32)
        s = np.ascontiguousarray(Ws, np.uint8).copy()
        l = np.ascontiguousarray(Wl, dt).copy()
        getattr(self._L, "or_lf_store_half" + sfx)(l.size, _p(s), _p(l))
        return s, l

    def lf_decode_batch_pmf(self, pmf, max_iters: int, mode: int = EXACT, early_stop: bool = True,
                            nthreads: int | None = None, f32: bool = False, want_soft: bool = False,
                            want_post: bool = False):
        """Decode F frames from symbol-level channel pmfs (float32 [F][N][q]); outputs as lf_decode_batch."""
        return self._decode_batch(pmf, True, max_iters, mode, early_stop, want_soft, want_post, nthreads, f32)

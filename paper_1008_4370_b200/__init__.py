"""B200-native batched Log-Fourier SP decoder for (2,k)-regular non-binary LDPC codes (arXiv:1008.4370).

Thin Python binding over the C-ABI library ``lib/libnbldpc.so`` (``include/nbldpc.h``).
This module only marshals arguments: every step of the decoding path runs in the
sm_100a kernels of ``csrc/``.  PyTorch supplies device memory and streams.  There is
no CPU fallback: if the library is missing or fails to load, importing the decoder
raises.
"""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np

from . import build as _build

__all__ = ["Code", "NbldpcError", "lib", "header_symbols", "FLOOR_LOG2"]

FLOOR_LOG2 = 200.0  # -log2 of a "zero" message entry (ex2 flushes it to 0)
_HERE = os.path.dirname(os.path.abspath(__file__))
_HEADER = os.path.join(os.path.dirname(_HERE), "include", "nbldpc.h")
_LIB = None

NBLDPC_OK = 0
VN_SEPARABLE, VN_DIRECT = 0, 1             # nbldpc_vn_algorithm_t
ALG_LOG_FOURIER, ALG_LOG_SP = 0, 1        # nbldpc_algorithm_t
MSG_F32, MSG_F16 = 0, 1                    # nbldpc_message_format_t
_STATUS = {0: "ok", -1: "invalid argument", -2: "not primitive", -3: "unsupported", -4: "CUDA error",
           -5: "out of memory"}


class NbldpcError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: nbldpc status {status} ({_STATUS.get(status, '?')})")
        self.status = status


class _Opts(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_size_t), ("syndrome_mode", ctypes.c_int), ("no_early_stop", ctypes.c_int),
                ("soft_out", ctypes.c_void_p), ("events_out", ctypes.c_void_p), ("slots", ctypes.c_int),
                ("use_graph", ctypes.c_int), ("vn_algorithm", ctypes.c_int), ("symbol_post_out", ctypes.c_void_p),
                ("symbol_map_out", ctypes.c_void_p), ("algorithm", ctypes.c_int), ("message_format", ctypes.c_int),
                ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t)]


def header_symbols() -> list[str]:
    """Function names declared in include/nbldpc.h."""
    txt = open(_HEADER).read()
    return sorted(set(re.findall(r"\b(nbldpc_[a-z_]+)\s*\(", txt)))


def lib():
    """Load (building with nvcc if the .so is absent or stale and nvcc exists) the C-ABI library."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = _build.LIB
    if os.path.exists(_build.NVCC):
        path = _build.build()
    if not os.path.exists(path):
        raise ImportError(f"libnbldpc.so not found at {path} and nvcc unavailable: the CUDA decoder is required")
    L = ctypes.CDLL(path)
    vp, i32, u32, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32, ctypes.c_size_t
    sig = {
        "nbldpc_code_create": (i32, [i32, u32, i32, i32, i32, vp, vp, vp, ctypes.POINTER(vp)]),
        "nbldpc_destroy": (None, [vp]),
        "nbldpc_status_string": (ctypes.c_char_p, [i32]),
        "nbldpc_last_cuda_error": (ctypes.c_char_p, []),
        "nbldpc_code_info": (i32, [vp, vp, vp, vp, vp, vp]),
        "nbldpc_slot_bytes": (sz, [vp]),
        "nbldpc_workspace_bytes": (sz, [vp, i32]),
        "nbldpc_last_decode_launches": (i32, [vp, ctypes.POINTER(ctypes.c_longlong)]),
        "nbldpc_decode": (i32, [vp, vp, i32, i32, vp, vp, vp, vp]),
        "nbldpc_decode_ex": (i32, [vp, vp, i32, i32, vp, vp, vp, vp, ctypes.POINTER(_Opts)]),
        "nbldpc_decode_host": (i32, [vp, vp, i32, i32, vp, vp, vp, vp, ctypes.POINTER(_Opts)]),
        "nbldpc_decode_pmf": (i32, [vp, vp, i32, i32, vp, vp, vp, vp, ctypes.POINTER(_Opts)]),
        "nbldpc_decode_pmf_host": (i32, [vp, vp, i32, i32, vp, vp, vp, vp, ctypes.POINTER(_Opts)]),
        "nbldpc_step": (i32, [vp, vp, i32, i32, vp, vp, vp, vp, vp, i32, vp]),
        "nbldpc_step_pmf": (i32, [vp, vp, i32, i32, vp, vp, vp, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = L
    return L


def _check(st: int, where: str):
    if st != NBLDPC_OK:
        detail = ""
        if st in (-4, -5):
            detail = " [" + lib().nbldpc_last_cuda_error().decode() + "]"
        raise NbldpcError(st, where + detail)


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream) -> int | None:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class Code:
    """A non-binary LDPC code on the current CUDA device (nbldpc_code_create)."""

    def __init__(self, m: int, poly: int, M: int, N: int, rows, cols, coeffs):
        L = lib()
        r = np.ascontiguousarray(rows, np.int32)
        c = np.ascontiguousarray(cols, np.int32)
        h = np.ascontiguousarray(coeffs, np.uint16)
        if not (r.size == c.size == h.size):
            raise ValueError("rows, cols, coeffs must have equal length")
        hnd = ctypes.c_void_p()
        st = L.nbldpc_code_create(int(m), int(poly), int(M), int(N), int(r.size), r.ctypes.data, c.ctypes.data,
                                  h.ctypes.data, ctypes.byref(hnd))
        _check(st, "nbldpc_code_create")
        self._h = hnd
        self._L = L
        self.m, self.q, self.M, self.N, self.E = m, 1 << m, M, N, int(r.size)
        kmax = ctypes.c_int()
        L.nbldpc_code_info(self._h, None, None, None, None, ctypes.byref(kmax))
        self.k_max = kmax.value

    def close(self):
        if getattr(self, "_h", None):
            self._L.nbldpc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def last_decode_launches(self) -> int:
        """Kernels launched by the most recent decode (synchronises its stream)."""
        n = ctypes.c_longlong()
        _check(self._L.nbldpc_last_decode_launches(self._h, ctypes.byref(n)), "nbldpc_last_decode_launches")
        return int(n.value)

    @property
    def slot_bytes(self) -> int:
        return int(self._L.nbldpc_slot_bytes(self._h))

    def workspace_bytes(self, frames: int) -> int:
        """Device bytes of the workspace a default decode of ``frames`` frames keeps (nbldpc_workspace_bytes)."""
        return int(self._L.nbldpc_workspace_bytes(self._h, int(frames)))

    def _opts(self, syndrome_mode=0, early_stop=True, soft=None, events=None, slots=0, use_graph=0, vn_algorithm=0,
              post=None, xmap=None, algorithm=0, message_format=0, workspace=None):
        o = _Opts()
        o.struct_size = ctypes.sizeof(_Opts)
        o.syndrome_mode = int(syndrome_mode)
        o.no_early_stop = 0 if early_stop else 1
        o.soft_out = _ptr(soft)
        o.events_out = _ptr(events)
        o.slots = int(slots)
        o.use_graph = int(use_graph)
        o.vn_algorithm = int(vn_algorithm)
        o.symbol_post_out = _ptr(post)
        o.symbol_map_out = _ptr(xmap)
        o.algorithm = int(algorithm)
        o.message_format = int(message_format)
        if workspace is not None:
            o.workspace = workspace.data_ptr()
            o.workspace_bytes = workspace.numel() * workspace.element_size()
        return o

    def _outputs(self, F, dev, want_soft, want_events, want_post):
        import torch

        out = {"hard": torch.empty((F, self.N), dtype=torch.uint8, device=dev),
               "ok": torch.empty(F, dtype=torch.uint8, device=dev),
               "iters": torch.empty(F, dtype=torch.int32, device=dev)}
        if want_soft:
            out["soft"] = torch.empty((F, self.N * self.m), dtype=torch.float32, device=dev)
        if want_events:
            out["events"] = torch.empty(F, dtype=torch.int32, device=dev)
        if want_post:
            out["post"] = torch.empty((F, self.N, self.q), dtype=torch.float32, device=dev)
            out["map"] = torch.empty((F, self.N), dtype=torch.uint8, device=dev)
        return out

    def decode(self, llr, max_iters: int, *, syndrome_mode: int = 0, early_stop: bool = True, want_soft=False,
               want_events=False, want_post=False, slots: int = 0, use_graph: int = 0, vn_algorithm: int = 0, out=None,
               stream=None, algorithm: int = 0, message_format: int = 0, workspace=None):
        """Decode frames. ``llr``: CUDA float32 tensor [F, N*m].  Returns a dict of CUDA tensors
        (hard uint8 [F,N], ok uint8 [F], iters int32 [F], optional soft float32 [F,N*m], events int32 [F],
        post float32 [F,N,q] symbol posterior and map uint8 [F,N] symbol-MAP decision).
        ``workspace``: optional caller-owned CUDA tensor of >= workspace_bytes(F) bytes (256-byte aligned)."""
        import torch

        if not (llr.is_cuda and llr.dtype == torch.float32 and llr.is_contiguous()):
            raise ValueError("llr must be a contiguous CUDA float32 tensor")
        F = llr.numel() // (self.N * self.m)
        if F * self.N * self.m != llr.numel() or F < 1:
            raise ValueError("llr size is not a multiple of N*m")
        if out is None:
            out = self._outputs(F, llr.device, want_soft, want_events, want_post)
        o = self._opts(syndrome_mode, early_stop, out.get("soft"), out.get("events"), slots, use_graph, vn_algorithm,
                       out.get("post"), out.get("map"), algorithm, message_format, workspace)
        st = self._L.nbldpc_decode_ex(self._h, llr.data_ptr(), F, int(max_iters), out["hard"].data_ptr(),
                                      out["ok"].data_ptr(), out["iters"].data_ptr(), _stream(stream),
                                      ctypes.byref(o))
        _check(st, "nbldpc_decode_ex")
        return out

    def decode_pmf(self, pmf, max_iters: int, *, syndrome_mode: int = 0, early_stop: bool = True, want_soft=False,
                   want_events=False, want_post=False, slots: int = 0, use_graph: int = 0, vn_algorithm: int = 0,
                   out=None, stream=None, algorithm: int = 0, message_format: int = 0):
        """Decode frames from symbol-level channel pmfs (nbldpc_decode_pmf).
        ``pmf``: CUDA float32 tensor [F, N, q] (any positive scale per row).  Same outputs as decode."""
        import torch

        if not (pmf.is_cuda and pmf.dtype == torch.float32 and pmf.is_contiguous()):
            raise ValueError("pmf must be a contiguous CUDA float32 tensor")
        F = pmf.numel() // (self.N * self.q)
        if F * self.N * self.q != pmf.numel() or F < 1:
            raise ValueError("pmf size is not a multiple of N*q")
        if out is None:
            out = self._outputs(F, pmf.device, want_soft, want_events, want_post)
        o = self._opts(syndrome_mode, early_stop, out.get("soft"), out.get("events"), slots, use_graph, vn_algorithm,
                       out.get("post"), out.get("map"), algorithm, message_format)
        st = self._L.nbldpc_decode_pmf(self._h, pmf.data_ptr(), F, int(max_iters), out["hard"].data_ptr(),
                                       out["ok"].data_ptr(), out["iters"].data_ptr(), _stream(stream),
                                       ctypes.byref(o))
        _check(st, "nbldpc_decode_pmf")
        return out

    def decode_host(self, llr_host, max_iters: int, *, syndrome_mode: int = 0, slots: int = 0, use_graph: int = 0,
                    vn_algorithm: int = 0, out=None, stream=None, algorithm: int = 0, message_format: int = 0):
        """End-to-end decode from HOST memory (pinned torch tensor or numpy array) to host outputs."""
        import torch

        if isinstance(llr_host, np.ndarray):
            llr_host = torch.from_numpy(np.ascontiguousarray(llr_host, np.float32))
        if llr_host.is_cuda or llr_host.dtype != torch.float32 or not llr_host.is_contiguous():
            raise ValueError("llr_host must be a contiguous host float32 tensor")
        F = llr_host.numel() // (self.N * self.m)
        if out is None:
            pin = llr_host.is_pinned()
            out = {"hard": torch.empty((F, self.N), dtype=torch.uint8, pin_memory=pin),
                   "ok": torch.empty(F, dtype=torch.uint8, pin_memory=pin),
                   "iters": torch.empty(F, dtype=torch.int32, pin_memory=pin)}
        o = self._opts(syndrome_mode, True, None, None, slots, use_graph, vn_algorithm, algorithm=algorithm,
                       message_format=message_format)
        st = self._L.nbldpc_decode_host(self._h, llr_host.data_ptr(), F, int(max_iters), out["hard"].data_ptr(),
                                        out["ok"].data_ptr(), out["iters"].data_ptr(), _stream(stream),
                                        ctypes.byref(o))
        _check(st, "nbldpc_decode_host")
        return out

    def decode_pmf_host(self, pmf_host, max_iters: int, *, slots: int = 0, vn_algorithm: int = 0, out=None,
                        stream=None, algorithm: int = 0):
        """End-to-end pmf decode from HOST memory (nbldpc_decode_pmf_host): pmf_host float32 [F, N, q]."""
        import torch

        if isinstance(pmf_host, np.ndarray):
            pmf_host = torch.from_numpy(np.ascontiguousarray(pmf_host, np.float32))
        if pmf_host.is_cuda or pmf_host.dtype != torch.float32 or not pmf_host.is_contiguous():
            raise ValueError("pmf_host must be a contiguous host float32 tensor")
        F = pmf_host.numel() // (self.N * self.q)
        if F * self.N * self.q != pmf_host.numel() or F < 1:
            raise ValueError("pmf size is not a multiple of N*q")
        if out is None:
            pin = pmf_host.is_pinned()
            out = {"hard": torch.empty((F, self.N), dtype=torch.uint8, pin_memory=pin),
                   "ok": torch.empty(F, dtype=torch.uint8, pin_memory=pin),
                   "iters": torch.empty(F, dtype=torch.int32, pin_memory=pin)}
        o = self._opts(0, True, None, None, slots, 0, vn_algorithm, algorithm=algorithm)
        st = self._L.nbldpc_decode_pmf_host(self._h, pmf_host.data_ptr(), F, int(max_iters), out["hard"].data_ptr(),
                                            out["ok"].data_ptr(), out["iters"].data_ptr(), _stream(stream),
                                            ctypes.byref(o))
        _check(st, "nbldpc_decode_pmf_host")
        return out

    def step(self, llr, iter_: int, w_in=None, want_u=False, want_soft=False, vn_algorithm: int = 0, stream=None):
        """One Log-Fourier iteration from state W^(iter) (parity tests).  Tensors in the packed
        -log2|x| + sign-bit format, [F, E, q]."""
        import torch

        F = llr.numel() // (self.N * self.m)
        dev = llr.device
        w_out = torch.empty((F, self.E, self.q), dtype=torch.float32, device=dev)
        u_out = torch.empty_like(w_out) if want_u else None
        hard = torch.empty((F, self.N), dtype=torch.uint8, device=dev)
        soft = torch.empty((F, self.N * self.m), dtype=torch.float32, device=dev) if want_soft else None
        st = self._L.nbldpc_step(self._h, llr.data_ptr(), F, int(iter_), _ptr(w_in), w_out.data_ptr(), _ptr(u_out),
                                 hard.data_ptr(), _ptr(soft), int(vn_algorithm), _stream(stream))
        _check(st, "nbldpc_step")
        return {"w": w_out, "u": u_out, "hard": hard, "soft": soft}

    def step_pmf(self, pmf, iter_: int, w_in=None, want_u=False, want_soft=False, stream=None):
        """nbldpc_step from symbol pmfs [F, N, q] (the cluster kernel's pmf variant; parity tests)."""
        import torch

        F = pmf.numel() // (self.N * self.q)
        dev = pmf.device
        w_out = torch.empty((F, self.E, self.q), dtype=torch.float32, device=dev)
        u_out = torch.empty_like(w_out) if want_u else None
        hard = torch.empty((F, self.N), dtype=torch.uint8, device=dev)
        soft = torch.empty((F, self.N * self.m), dtype=torch.float32, device=dev) if want_soft else None
        st = self._L.nbldpc_step_pmf(self._h, pmf.data_ptr(), F, int(iter_), _ptr(w_in), w_out.data_ptr(), _ptr(u_out),
                                     hard.data_ptr(), _ptr(soft), _stream(stream))
        _check(st, "nbldpc_step_pmf")
        return {"w": w_out, "u": u_out, "hard": hard, "soft": soft}

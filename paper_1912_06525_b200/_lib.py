"""ctypes binding of libkatzb200.so (the C-ABI declared in include/katzb200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_1912_06525_b200/csrc``).  There is no fallback: if the
library or a CUDA device is missing, every device entry point raises
``KatzDeviceError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# KZ_LIB_PATH: an alternative build of the same library (kernel experiments)
LIB_PATH = os.environ.get("KZ_LIB_PATH") or os.path.join(_HERE, "libkatzb200.so")

KZ_OK = 0
KZ_EARG = 1
KZ_ENOTSPD = 2
KZ_ESPECTRUM = 3
KZ_ECUDA = 4
KZ_EOOM = 5

HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "katzb200.h")


def header_symbols(path=HEADER_PATH):
    """Names of the functions include/katzb200.h declares."""
    import re

    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", " ", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kz_[a-z0-9_]+)\s*\(", text)))


class KatzDeviceError(RuntimeError):
    """The CUDA extension or the GPU is unavailable (there is no CPU path)."""


class KzReport(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int64),
        ("converged", ctypes.c_int32),
        ("status", ctypes.c_int32),
        ("final_residual_norm", ctypes.c_double),
        ("rhs_norm", ctypes.c_double),
    ]


class KzCgArgs(ctypes.Structure):
    _fields_ = [
        ("b", ctypes.c_int32),
        ("clamp", ctypes.c_int32),
        ("qpos", ctypes.POINTER(ctypes.c_int64)),
        ("rhs", ctypes.c_void_p),
        ("beta", ctypes.c_double),
        ("tol", ctypes.c_double),
        ("max_iter", ctypes.c_int64),
        ("x0", ctypes.c_void_p),
        ("perm", ctypes.c_void_p),
        ("scores", ctypes.c_void_p),
        ("reports", ctypes.POINTER(KzReport)),
        ("device_ms", ctypes.POINTER(ctypes.c_float)),
    ]


class KzTopkArgs(ctypes.Structure):
    _fields_ = [
        ("b", ctypes.c_int32),
        ("k", ctypes.c_int32),
        ("n", ctypes.c_int64),
        ("scores", ctypes.c_void_p),
        ("mask_graph", ctypes.c_void_p),
        ("mask_rows", ctypes.POINTER(ctypes.c_int64)),
        ("self_ids", ctypes.POINTER(ctypes.c_int64)),
        ("ids_out", ctypes.c_void_p),
        ("vals_out", ctypes.c_void_p),
        ("count_out", ctypes.c_void_p),
        ("bound_vals", ctypes.c_void_p),
        ("bound_ids", ctypes.c_void_p),
    ]


class KzLrcDesc(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("n1", ctypes.c_int64),
        ("n2", ctypes.c_int64),
        ("ell", ctypes.c_int64),
        ("beta", ctypes.c_double),
        ("full", ctypes.c_void_p),
        ("a12", ctypes.c_void_p),
        ("a21", ctypes.c_void_p),
        ("a22", ctypes.c_void_p),
        ("minv", ctypes.c_void_p),
        ("linv", ctypes.c_void_p),
        ("linvT", ctypes.c_void_p),
        ("u", ctypes.c_void_p),
        ("udT", ctypes.c_void_p),
        ("sigma", ctypes.POINTER(ctypes.c_double)),
    ]


class KzLrcArgs(ctypes.Structure):
    _fields_ = [
        ("b", ctypes.c_int32),
        ("chunk", ctypes.c_int32),
        ("clamp", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
        ("qpos", ctypes.POINTER(ctypes.c_int64)),
        ("f", ctypes.c_void_p),
        ("tol", ctypes.c_double),
        ("max_iter", ctypes.c_int64),
        ("x0", ctypes.c_void_p),
        ("perm", ctypes.c_void_p),
        ("out", ctypes.c_void_p),
        ("reports", ctypes.POINTER(KzReport)),
        ("device_ms", ctypes.POINTER(ctypes.c_float)),
    ]


class KzEigenDesc(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("r", ctypes.c_int64),
        ("ldr", ctypes.c_int64),
        ("beta", ctypes.c_double),
        ("op", ctypes.c_void_p),
        ("u", ctypes.c_void_p),
        ("au", ctypes.c_void_p),
        ("w", ctypes.c_void_p),
        ("a2u", ctypes.c_void_p),
        ("a3u", ctypes.c_void_p),
        ("a4u", ctypes.c_void_p),
    ]


_lock = threading.Lock()
_lib = None
CHECKED = False  # a checked build (KZ_CHECKED) is loaded: poisoned workspaces, red-zone checks


def load(require=True):
    """Load libkatzb200.so once; raises KatzDeviceError if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            if require:
                raise KatzDeviceError(
                    f"{LIB_PATH} is missing; build it with __graft_entry__.build() "
                    "(there is no CPU fallback)"
                )
            return None
        lib = ctypes.CDLL(LIB_PATH)
        _declare(lib)
        global CHECKED
        CHECKED = bool(lib.kz_checked())
        _lib = lib
        return lib


def _declare(lib):
    c = ctypes
    vp, i32, i64, dbl, sz = c.c_void_p, c.c_int32, c.c_int64, c.c_double, c.c_size_t
    lib.kz_last_error.restype = c.c_char_p
    lib.kz_version.restype = c.c_int
    lib.kz_launch_count.restype = c.c_longlong
    lib.kz_num_sms.restype = c.c_int
    lib.kz_checked.restype = c.c_int
    lib.kz_checked_redzones.argtypes = [c.c_void_p, c.POINTER(c.c_int64), c.c_int64]
    lib.kz_checked_redzones.restype = c.c_int64
    lib.kz_k1_timing.argtypes = [c.c_int]
    lib.kz_k1_timing_read.argtypes = [c.POINTER(c.c_double), c.POINTER(c.c_longlong)]
    lib.kz_graph_create.argtypes = [i64, i64, i64, vp, vp, c.POINTER(vp)]
    lib.kz_graph_destroy.argtypes = [vp]
    lib.kz_graph_info.argtypes = [vp] + [c.POINTER(i64)] * 5
    lib.kz_spmm_workspace_bytes.argtypes = [vp, i32, i32]
    lib.kz_spmm_workspace_bytes.restype = sz
    lib.kz_spmm.argtypes = [vp, i32, i32, vp, vp, vp, vp, dbl, dbl, dbl, vp, vp, vp, sz, vp]
    lib.kz_cg_workspace_bytes.argtypes = [vp, i32]
    lib.kz_cg_workspace_bytes.restype = sz
    lib.kz_cg_batch.argtypes = [vp, c.POINTER(KzCgArgs), vp, sz, vp]
    lib.kz_topk_workspace_bytes.argtypes = [i32, i64, i32]
    lib.kz_topk_workspace_bytes.restype = sz
    lib.kz_topk_batch.argtypes = [c.POINTER(KzTopkArgs), vp, sz, vp]
    lib.kz_coldot.argtypes = [i64, i32, vp, vp, vp, vp, sz, vp]
    lib.kz_coldot_workspace_bytes.argtypes = [i64, i32]
    lib.kz_coldot_workspace_bytes.restype = sz
    lib.kz_vec_op.argtypes = [i32, i64, dbl, vp, dbl, vp, vp, vp]
    lib.kz_profile_gather.argtypes = [vp, i64, i32, vp, vp, vp, i32, vp, i32, vp]
    lib.kz_pearson_rerank.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, vp, vp, vp]
    lib.kz_graph_create_weighted.argtypes = [i64, i64, i64, vp, vp, vp, c.POINTER(vp)]
    lib.kz_connected_components.argtypes = [i64, i64, vp, vp, vp, vp]
    lib.kz_edges_to_csr_workspace_bytes.argtypes = [i64, i64]
    lib.kz_edges_to_csr_workspace_bytes.restype = sz
    lib.kz_edges_to_csr.argtypes = [i64, i64, vp, vp, vp, vp, vp, c.POINTER(c.c_int64), vp, sz, vp]
    lib.kz_lrc_create.argtypes = [c.POINTER(KzLrcDesc), c.POINTER(vp)]
    lib.kz_lrc_destroy.argtypes = [vp]
    lib.kz_lrc_info.argtypes = [vp, c.POINTER(i64), c.POINTER(i64), c.POINTER(i64), c.POINTER(i64)]
    lib.kz_lrc_workspace_bytes.argtypes = [vp, i32, i32]
    lib.kz_lrc_workspace_bytes.restype = sz
    lib.kz_lrc_batch.argtypes = [vp, c.POINTER(KzLrcArgs), vp, sz, vp]
    lib.kz_lrc_apply.argtypes = [vp, i32, i32, vp, vp, vp, vp, sz, vp]
    pi64 = c.POINTER(i64)
    lib.kz_partition.argtypes = [i64, vp, vp, i64, i64, vp, vp, pi64, pi64, pi64]
    lib.kz_min_degree_order.argtypes = [i64, vp, vp, vp]
    lib.kz_min_degree_orders.argtypes = [i64, vp, vp, vp, vp]
    lib.kz_eigen_create.argtypes = [c.POINTER(KzEigenDesc), c.POINTER(vp)]
    lib.kz_eigen_destroy.argtypes = [vp]
    lib.kz_eigen_workspace_bytes.argtypes = [vp, i32]
    lib.kz_eigen_workspace_bytes.restype = sz
    lib.kz_eigen_batch.argtypes = [vp, c.POINTER(KzCgArgs), vp, sz, vp]


def error_from_status(code, lib=None):
    """Map a KZ_* status to the reference's exception types."""
    lib = lib or _lib
    msg = lib.kz_last_error().decode() if lib is not None else ""
    if code == KZ_EARG:
        return ValueError(msg)
    if code == KZ_ENOTSPD:
        return RuntimeError(msg or "operator is not positive definite")
    if code == KZ_ESPECTRUM:
        from .factor import SpectrumError

        return SpectrumError(msg)
    if code == KZ_EOOM:
        return MemoryError(msg)
    return KatzDeviceError(msg or f"CUDA failure (status {code})")


def check(code):
    if code != KZ_OK:
        Workspace._tls.pending = []
        raise error_from_status(code)
    if CHECKED:
        Workspace.verify_redzones()


def torch_cuda():
    """Import torch and insist on a CUDA device (no CPU fallback)."""
    import torch

    if not torch.cuda.is_available():
        raise KatzDeviceError("no CUDA device: the B200 query path has no CPU fallback")
    return torch


def stream_ptr(torch):
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def coldot(torch, lib, x, y, out, n, b=1, stream=None):
    """out[j] = X[:, j] . Y[:, j] (kz_coldot) with this thread's scratch."""
    ws = Workspace.get(torch, lib.kz_coldot_workspace_bytes(n, b), slot="coldot")
    check(lib.kz_coldot(n, b, ptr(x), ptr(y), ptr(out), ptr(ws), ws.numel(),
                        stream if stream is not None else stream_ptr(torch)))


def vec_op(torch, lib, op, n, a, x, b, y, out):
    """kz_vec_op: op 0 out = a*x + b*y (separately rounded), op 1 out = x / a."""
    check(lib.kz_vec_op(op, n, float(a), ptr(x), float(b), ptr(y), ptr(out), stream_ptr(torch)))


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def i64_array(values):
    arr = np.ascontiguousarray(values, dtype=np.int64)
    return arr, arr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


class Workspace:
    """Per-thread cache of device scratch buffers (grown on demand)."""

    _tls = threading.local()

    @classmethod
    def get(cls, torch, nbytes, slot="default"):
        cache = getattr(cls._tls, "cache", None)
        if cache is None:
            cache = cls._tls.cache = {}
        buf = cache.get(slot)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device="cuda")
            cache[slot] = buf
        if CHECKED:
            # poison (NaN doubles, -1 ints) and remember it for the red-zone check
            buf.fill_(0xFF)
            pend = getattr(cls._tls, "pending", None)
            if pend is None:
                pend = cls._tls.pending = []
            pend.append(buf)
        return buf

    @classmethod
    def verify_redzones(cls):
        """Checked builds: every red zone the library carved in the pending
        workspaces still holds the 0xFF poison (no slice overran)."""
        pend = getattr(cls._tls, "pending", None) or []
        cls._tls.pending = []
        if not pend:
            return
        import torch

        lib = load()
        for buf in pend:
            cap = 1 << 16
            offs = np.zeros(cap, dtype=np.int64)
            k = lib.kz_checked_redzones(ctypes.c_void_p(buf.data_ptr()), offs.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), cap)
            if k == 0:
                continue
            o = torch.as_tensor(offs[: min(k, cap)], device=buf.device)
            idx = (o[:, None] + torch.arange(256, device=buf.device)[None, :]).reshape(-1)
            idx = idx[idx < buf.numel()]
            bad = int((buf[idx] != 0xFF).sum().item())
            if bad:
                raise RuntimeError(f"checked build: {bad} red-zone bytes overwritten in a workspace")

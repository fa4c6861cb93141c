"""paper_1804_10694_b200 -- B200-native fp32 GEMM (the Tiramisu paper's sgemm).

Thin ctypes binding over the C ABI in ``include/tm.h`` (``_lib/libtm.so``).
Argument marshalling only: every step of the computation runs in the CUDA
kernels of the library.  torch is used for device memory, streams and process
groups.  There is no CPU fallback: if the library is missing this module
raises at import.

    C = alpha * A @ B + beta * C
"""
from __future__ import annotations

import ctypes
import os

__all__ = [
    "ALGO_AUTO", "ALGO_TF32X3", "ALGO_SIMT_F32", "ALGO_TF32X1", "ALGO_BF16X9", "TmError", "lib", "lib_path", "sgemm",
    "sgemm_ex", "sgemm_host", "plan_name", "plan_config", "tune", "tune_cache_save", "tune_cache_load",
    "tune_cache_clear", "tune_cache_size", "dist_rows", "Comm", "CeComm", "blur", "blur_dist_loopback", "status_string", "EXPORTED_SYMBOLS",
]

ALGO_AUTO, ALGO_TF32X3, ALGO_SIMT_F32, ALGO_TF32X1, ALGO_BF16X9 = 0, 1, 2, 3, 4

_PKG = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(_PKG, "_lib", "libtm.so")
# Tests only (tests/test_product_mutants.py): load a mutant build instead.
lib_path = os.environ.get("TM_LIB_PATH", lib_path)

# Every function include/tm.h declares (checked by tests/test_abi.py).
EXPORTED_SYMBOLS = [
    "tm_sgemm", "tm_sgemm_ex", "tm_sgemm_op", "tm_sgemm_colmajor", "tm_conv2d_nhwc", "tm_sgemm_host", "tm_release_workspace", "tm_status_string", "tm_get_version",
    "tm_sgemm_plan_name", "tm_comm_get_unique_id", "tm_comm_init", "tm_comm_destroy", "tm_comm_rank",
    "tm_dist_rows", "tm_dist_chunk", "tm_sgemm_dist", "tm_sgemm_dist_fused", "tm_sgemm_dist_loopback", "tm_sgemm_dist_allgather", "tm_comm_check", "tm_comm_bytes_received",
    "tm_sgemm_tune", "tm_tune_cache_size", "tm_tune_cache_clear", "tm_tune_cache_save", "tm_tune_cache_load",
    "tm_sgemm_plan_config", "tm_sgemm_streamk_region", "tm_blur", "tm_blur_dist", "tm_blur_dist_loopback",
    "tm_sgemm_summa", "tm_summa_panel", "tm_sgemm_summa_loopback", "tm_conv2d_plan_name",
    "tm_ipc_export", "tm_ce_create", "tm_ce_connect", "tm_ce_destroy", "tm_ce_bytes_received", "tm_sgemm_dist_ce",
]


class TmError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {status_string(status)} ({status})")


def _load():
    if not os.path.exists(lib_path):
        raise ImportError(
            f"{lib_path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(lib_path)
    i64, f32, vp, ci = ctypes.c_int64, ctypes.c_float, ctypes.c_void_p, ctypes.c_int
    gemm = [i64, i64, i64, f32, vp, i64, vp, i64, f32, vp, i64, vp]
    L.tm_sgemm.argtypes = gemm
    L.tm_sgemm_ex.argtypes = gemm + [ci]
    L.tm_sgemm_host.argtypes = gemm + [ci]
    L.tm_sgemm_op.argtypes = [ci, ci] + gemm + [ci]
    L.tm_sgemm_colmajor.argtypes = [ctypes.c_char, ctypes.c_char] + gemm
    L.tm_conv2d_nhwc.argtypes = [i64] * 8 + [f32, vp, vp, f32, vp, vp, ci]
    L.tm_sgemm_plan_name.argtypes = [i64, i64, i64, f32, vp, i64, vp, i64, f32, vp, i64, ci]
    L.tm_sgemm_plan_name.restype = ctypes.c_char_p
    L.tm_status_string.argtypes = [ci]
    L.tm_status_string.restype = ctypes.c_char_p
    L.tm_dist_rows.argtypes = [i64, ci, ci, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.tm_sgemm_streamk_region.argtypes = [i64, i64, ci, ci, ctypes.POINTER(i64), ctypes.POINTER(ci)]
    L.tm_dist_chunk.argtypes = [i64, ci, ci, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.tm_comm_get_unique_id.argtypes = [vp]
    L.tm_comm_init.argtypes = [ctypes.POINTER(vp), ci, ci, vp]
    L.tm_comm_destroy.argtypes = [vp]
    L.tm_comm_rank.argtypes = [vp, ctypes.POINTER(ci), ctypes.POINTER(ci)]
    L.tm_comm_check.argtypes = [vp, ci]
    L.tm_comm_bytes_received.argtypes = [vp, ctypes.POINTER(ctypes.c_uint64)]
    L.tm_sgemm_dist.argtypes = [vp, i64, i64, i64, f32, vp, i64, vp, i64, ci, f32, vp, i64, vp]
    L.tm_sgemm_dist_fused.argtypes = [vp, i64, i64, i64, f32, vp, i64, vp, i64, ci, f32, vp, i64, vp]
    L.tm_sgemm_dist_loopback.argtypes = [ci, ci, ci, i64, i64, i64, f32, vp, i64, vp, i64, f32, vp, i64, vp, vp]
    L.tm_sgemm_dist_allgather.argtypes = [vp, i64, i64, i64, f32, vp, i64, vp, vp, i64, f32, vp, i64, vp]
    pi = ctypes.POINTER(ci)
    L.tm_sgemm_tune.argtypes = [ci, ci] + gemm + [ci, pi, pi, pi, ctypes.POINTER(f32)]
    L.tm_tune_cache_size.argtypes = []
    L.tm_tune_cache_clear.argtypes = []
    L.tm_tune_cache_save.argtypes = [ctypes.c_char_p]
    L.tm_tune_cache_load.argtypes = [ctypes.c_char_p]
    L.tm_sgemm_plan_config.argtypes = [ci, ci, i64, i64, i64, f32, vp, i64, vp, i64, f32, vp, i64, ci, pi, pi, pi, pi]
    L.tm_blur.argtypes = [i64, i64, vp, i64, vp, i64, vp]
    L.tm_blur_dist.argtypes = [vp, i64, i64, vp, i64, vp, i64, vp]
    L.tm_blur_dist_loopback.argtypes = [ci, i64, i64, vp, i64, vp, i64, vp, vp]
    L.tm_conv2d_plan_name.argtypes = [i64] * 8 + [f32, vp, vp, vp, ci]
    L.tm_conv2d_plan_name.restype = ctypes.c_char_p
    L.tm_sgemm_summa.argtypes = [vp, ci, ci, i64, i64, i64, f32, vp, i64, vp, i64, f32, vp, i64, vp]
    L.tm_summa_panel.argtypes = [i64, ci, ci, ci, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.tm_sgemm_summa_loopback.argtypes = [ci, ci, i64, i64, i64, f32, vp, vp, vp, vp, f32, vp, vp, vp, vp]
    L.tm_ipc_export.argtypes = [vp, vp]
    L.tm_ce_create.argtypes = [ctypes.POINTER(vp), ci, ci, vp]
    L.tm_ce_connect.argtypes = [vp, vp]
    L.tm_ce_destroy.argtypes = [vp]
    L.tm_ce_bytes_received.argtypes = [vp, ctypes.POINTER(ctypes.c_uint64)]
    L.tm_sgemm_dist_ce.argtypes = [vp, i64, i64, i64, f32, vp, i64, vp, i64, vp, ci, f32, vp, i64, ci, vp]
    for name in EXPORTED_SYMBOLS:
        fn = getattr(L, name)
        if fn.restype is ctypes.c_int or name in ("tm_status_string", "tm_sgemm_plan_name", "tm_conv2d_plan_name"):
            continue
        fn.restype = ctypes.c_int
    return L


lib = _load()


def status_string(status: int) -> str:
    return lib.tm_status_string(int(status)).decode()


def _check(status: int, what: str):
    if status != 0:
        raise TmError(status, what)


def _ld(t) -> int:
    """Leading dimension (elements) of a row-major 2-D view with unit column stride."""
    sh = t.shape
    if len(sh) != 2:
        raise ValueError("expected a 2-D tensor")
    st = t.stride()
    if sh[1] > 1 and st[1] != 1:
        raise ValueError("expected unit column stride (row-major)")
    if sh[0] <= 1:
        return max(int(st[0]) if sh[0] == 1 else 1, int(sh[1]), 1)
    return int(st[0])


def _ptr(t):
    # ctypes converts a Python int (or None) for a c_void_p argument itself
    return None if t is None else t.data_ptr()


_raw_stream = None


def _stream(stream):
    """cudaStream_t (as an int) of `stream` (int / torch.cuda.Stream) or torch's current stream."""
    global _raw_stream
    if stream is not None:
        return int(getattr(stream, "cuda_stream", stream))
    if _raw_stream is None:
        import torch
        get = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        _raw_stream = (lambda: get(torch.cuda.current_device())) if get else \
            (lambda: torch.cuda.current_stream().cuda_stream)
    return _raw_stream()


_F32 = None


def _f32_dtype():
    import torch
    return torch.float32


def _f32(name, t):
    global _F32
    if t is None:
        return None
    if _F32 is None:
        import torch
        _F32 = torch.float32
    if t.dtype is not _F32:
        raise TypeError(f"{name} must be float32")
    return t


def _on_device(**tensors):
    """Every tensor is a CUDA tensor on the current device (a host or other-device
    pointer handed to a kernel would fault or poison the context)."""
    import torch
    for name, t in tensors.items():
        if t is not None and not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (got {t.device})")
    dev = torch.cuda.current_device()
    for name, t in tensors.items():
        if t is not None and t.device.index != dev:
            raise ValueError(f"{name} is on {t.device} but the current device is cuda:{dev}")


def _shape(name, t, rows, cols):
    if t is not None and (t.dim() != 2 or tuple(t.shape) != (rows, cols)):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected ({rows}, {cols})")


def sgemm_ex(A, B, C, alpha: float = 1.0, beta: float = 0.0, algo: int = ALGO_AUTO, stream=None,
             m=None, n=None, k=None):
    """In place: C <- alpha*A@B + beta*C on CUDA tensors (row-major 2-D views).

    A may be None when alpha == 0 or k == 0 (it is then not read), likewise B.
    Shapes must agree: A (m, k), B (k, n), C (m, n) -- ValueError otherwise, as
    for torch.mm -- and every tensor must live on the current CUDA device.
    """
    A, B, C = _f32("A", A), _f32("B", B), _f32("C", C)
    m = C.shape[0] if m is None else m
    n = C.shape[1] if n is None else n
    k = (A.shape[1] if A is not None else (B.shape[0] if B is not None else 0)) if k is None else k
    _shape("A", A, m, k)
    _shape("B", B, k, n)
    _shape("C", C, m, n)
    _on_device(A=A, B=B, C=C)
    lda = _ld(A) if A is not None else max(k, 1)
    ldb = _ld(B) if B is not None else max(n, 1)
    st = lib.tm_sgemm_ex(m, n, k, float(alpha), _ptr(A), lda, _ptr(B), ldb, float(beta), _ptr(C), _ld(C),
                         _stream(stream), int(algo))
    _check(st, "tm_sgemm_ex")
    return C


def sgemm_op(A, B, C, alpha: float = 1.0, beta: float = 0.0, opa: str = "N", opb: str = "N",
             algo: int = ALGO_AUTO, stream=None):
    """C <- alpha*op(A)@op(B) + beta*C; A, B given as stored (A is k x m when
    opa == "T", B is n x k when opb == "T"), row-major CUDA tensors."""
    A, B, C = _f32("A", A), _f32("B", B), _f32("C", C)
    m, n = C.shape
    ta, tb = opa == "T", opb == "T"
    k = A.shape[0] if ta else A.shape[1]
    _shape("A", A, *((k, m) if ta else (m, k)))
    _shape("B", B, *((n, k) if tb else (k, n)))
    _on_device(A=A, B=B, C=C)
    st = lib.tm_sgemm_op(int(ta), int(tb), m, n, k, float(alpha), _ptr(A), _ld(A), _ptr(B), _ld(B), float(beta),
                         _ptr(C), _ld(C), _stream(stream), int(algo))
    _check(st, "tm_sgemm_op")
    return C


def tune(A, B, C, alpha: float = 1.0, beta: float = 0.0, opa: str = "N", opb: str = "N", reps: int = 5,
         stream=None):
    """Time every tensor-core configuration on these operands (C is read, not
    written) and cache the fastest for this shape; later calls use it.
    Returns (cg, bn_cta, streamk, median_ms)."""
    A, B, C = _f32("A", A), _f32("B", B), _f32("C", C)
    m, n = C.shape
    ta, tb = opa == "T", opb == "T"
    k = A.shape[0] if ta else A.shape[1]
    _shape("A", A, *((k, m) if ta else (m, k)))
    _shape("B", B, *((n, k) if tb else (k, n)))
    _on_device(A=A, B=B, C=C)
    cg, bn, sk, ms = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_float()
    st = lib.tm_sgemm_tune(int(ta), int(tb), m, n, k, float(alpha), _ptr(A), _ld(A), _ptr(B), _ld(B), float(beta),
                           _ptr(C), _ld(C), _stream(stream), int(reps), ctypes.byref(cg), ctypes.byref(bn),
                           ctypes.byref(sk), ctypes.byref(ms))
    _check(st, "tm_sgemm_tune")
    return cg.value, bn.value, sk.value, ms.value


def plan_config(m, n, k, alpha=1.0, beta=0.0, A_ptr=1 << 40, lda=None, B_ptr=2 << 40, ldb=None, C_ptr=3 << 40,
                ldc=None, opa="N", opb="N", algo=ALGO_AUTO):
    """Host-only: (path, cg, bn_cta, streamk) tm_sgemm_op would use; path 3 =
    tensor cores, 4 = SIMT, 2 = scale, 1 = no-op, 0 = invalid.  The default
    pointers are 1 TiB apart, so no operand overlaps C at any size."""
    ta, tb = opa == "T", opb == "T"
    lda = (max(m, 1) if ta else max(k, 1)) if lda is None else lda
    ldb = (max(k, 1) if tb else max(n, 1)) if ldb is None else ldb
    ldc = max(n, 1) if ldc is None else ldc
    out = [ctypes.c_int() for _ in range(4)]
    lib.tm_sgemm_plan_config(int(ta), int(tb), m, n, k, float(alpha), ctypes.c_void_p(A_ptr), lda,
                             ctypes.c_void_p(B_ptr), ldb, float(beta), ctypes.c_void_p(C_ptr), ldc, int(algo),
                             *[ctypes.byref(o) for o in out])
    return tuple(o.value for o in out)


def tune_cache_save(path: str) -> None:
    _check(lib.tm_tune_cache_save(path.encode()), "tm_tune_cache_save")


def tune_cache_load(path: str) -> int:
    n = lib.tm_tune_cache_load(path.encode())
    if n < 0:
        raise OSError(f"cannot read {path}")
    return n


def tune_cache_clear() -> None:
    _check(lib.tm_tune_cache_clear(), "tm_tune_cache_clear")


def tune_cache_size() -> int:
    return lib.tm_tune_cache_size()


def conv2d_nhwc(X, Wt, Y, alpha: float = 1.0, beta: float = 0.0, pad: int = 0, algo: int = ALGO_AUTO, stream=None):
    """Y <- alpha * conv(X, Wt) + beta * Y: X (Nb, H, W, C) NHWC, Wt (F, R, S, C)
    KRSC, Y (Nb, Ho, Wo, F); dense float32 CUDA tensors, stride 1, zero padding."""
    for name, t in (("X", X), ("Wt", Wt), ("Y", Y)):
        _f32(name, t)
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
    _on_device(X=X, Wt=Wt, Y=Y)
    nb, h, w, c = X.shape
    f, r, s, c2 = Wt.shape
    if c2 != c or tuple(Y.shape) != (nb, h + 2 * pad - r + 1, w + 2 * pad - s + 1, f):
        raise ValueError("shape mismatch")
    st = lib.tm_conv2d_nhwc(nb, h, w, c, f, r, s, pad, float(alpha), _ptr(X), _ptr(Wt), float(beta), _ptr(Y),
                            _stream(stream), int(algo))
    _check(st, "tm_conv2d_nhwc")
    return Y


def conv2d_plan_name(nb, h, w, c, f, r, s, pad, alpha=1.0, algo=ALGO_AUTO, X_ptr=1 << 20, Wt_ptr=1 << 30,
                     Y_ptr=1 << 40) -> str:
    """Host-only: the kernel tm_conv2d_nhwc would run ("direct", "implicit_gemm", "simt", ...)."""
    return lib.tm_conv2d_plan_name(nb, h, w, c, f, r, s, pad, float(alpha), ctypes.c_void_p(X_ptr),
                                   ctypes.c_void_p(Wt_ptr), ctypes.c_void_p(Y_ptr), int(algo)).decode()


def sgemm(A, B, C, alpha: float = 1.0, beta: float = 0.0, stream=None):
    """C <- alpha*A@B + beta*C (AUTO path: 3xTF32 tensor cores when aligned)."""
    return sgemm_ex(A, B, C, alpha, beta, ALGO_AUTO, stream)


def plan_name(m, n, k, alpha=1.0, beta=0.0, A_ptr=0, lda=None, B_ptr=0, ldb=None, C_ptr=0, ldc=None,
              algo=ALGO_AUTO) -> str:
    """Host-only: the path tm_sgemm_ex would take (no device needed)."""
    lda = max(k, 1) if lda is None else lda
    ldb = max(n, 1) if ldb is None else ldb
    ldc = max(n, 1) if ldc is None else ldc
    return lib.tm_sgemm_plan_name(m, n, k, float(alpha), ctypes.c_void_p(A_ptr), lda, ctypes.c_void_p(B_ptr),
                                  ldb, float(beta), ctypes.c_void_p(C_ptr), ldc, int(algo)).decode()


def sgemm_host(A, B, C, alpha: float = 1.0, beta: float = 0.0, algo: int = ALGO_AUTO, stream=None):
    """End-to-end on HOST (CPU, ideally pinned) float32 tensors/arrays: copies in,
    computes on the current GPU, copies C back; synchronous."""
    import numpy as np

    def info(x):
        if x is None:
            return None, 0
        if isinstance(x, np.ndarray):
            if x.dtype != np.float32:
                raise TypeError("float32 required")
            if x.ndim != 2:
                raise ValueError("expected a 2-D array")
            # row-major views only: unit column stride, positive row stride
            if x.shape[1] > 1 and x.strides[1] != 4:
                raise ValueError("expected unit column stride (row-major)")
            if x.shape[0] > 1 and (x.strides[0] <= 0 or x.strides[0] % 4):
                raise ValueError("expected a positive row stride that is a multiple of 4 bytes")
            ld = x.strides[0] // 4 if x.shape[0] > 1 else max(x.shape[1], 1)
            return ctypes.c_void_p(x.ctypes.data), ld
        if x.is_cuda:
            raise ValueError("sgemm_host takes host buffers")
        if x.dtype != _f32_dtype():
            raise TypeError("float32 required")
        return ctypes.c_void_p(x.data_ptr()), _ld(x)

    m, n = C.shape
    k = A.shape[1] if A is not None else (B.shape[0] if B is not None else 0)
    for name, x, shp in (("A", A, (m, k)), ("B", B, (k, n))):
        if x is not None and tuple(x.shape) != shp:
            raise ValueError(f"{name} has shape {tuple(x.shape)}, expected {shp}")

    pa, lda = info(A)
    pb, ldb = info(B)
    pc, ldc = info(C)
    st = lib.tm_sgemm_host(m, n, k, float(alpha), pa, lda or max(k, 1), pb, ldb or max(n, 1), float(beta), pc,
                           ldc, _stream(stream), int(algo))
    _check(st, "tm_sgemm_host")
    return C


def streamk_region(num_tiles: int, kblocks: int, clusters: int, mode: int = -1):
    """(sk_tiles, clusters_used) of a stream-K launch (tm_sgemm_streamk_region)."""
    sk, cu = ctypes.c_int64(), ctypes.c_int()
    _check(lib.tm_sgemm_streamk_region(num_tiles, kblocks, clusters, mode, ctypes.byref(sk), ctypes.byref(cu)),
           "tm_sgemm_streamk_region")
    return int(sk.value), int(cu.value)


def dist_rows(m: int, nranks: int, rank: int):
    r0, nr = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.tm_dist_rows(m, nranks, rank, ctypes.byref(r0), ctypes.byref(nr)), "tm_dist_rows")
    return r0.value, nr.value


def dist_chunks(k: int, nranks: int):
    """K-chunk schedule of the distributed broadcast: list of (k0, kr)."""
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.tm_dist_chunk(k, nranks, -1, ctypes.byref(a), ctypes.byref(b)), "tm_dist_chunk")
    out = []
    for i in range(a.value):
        _check(lib.tm_dist_chunk(k, nranks, i, ctypes.byref(a), ctypes.byref(b)), "tm_dist_chunk")
        out.append((a.value, b.value))
    return out


def sgemm_dist_loopback(m, n, k, A_locals, Bs, C_locals, alpha=1.0, beta=0.0, root=0, stream=None, allgather=False,
                        fused=False, transport="nccl"):
    """Single-process emulation of the row-sharded mode:
    len(A_locals) simulated ranks on the current GPU, same schedule as
    Comm.sgemm (or Comm.sgemm_allgather when allgather=True: Bs[r] holds rank
    r's k-row shard in place; or Comm.sgemm(fused=True)'s flag-gated single
    launch when fused=True).  transport="ce": the copy-engine transport MODEL
    (tm.h modes 3, 4: no data moves -- fill every Bs[r] with B first -- chunks
    are released on a link-rate schedule, GEMMs keep every SM but one).
    Returns the bytes each simulated rank received."""
    P = len(A_locals)
    arr = lambda ts: (ctypes.c_void_p * P)(*[t.data_ptr() for t in ts])
    lda = next((_ld(a) for a in A_locals if a.shape[0] > 0), max(k, 1))
    ldc = next((_ld(c) for c in C_locals if c.shape[0] > 0), max(n, 1))
    got = (ctypes.c_uint64 * P)()
    mode = 1 if allgather else (2 if fused else 0) + (2 if transport == "ce" else 0)
    st = lib.tm_sgemm_dist_loopback(P, int(root), mode, m, n, k, float(alpha), arr(A_locals), lda,
                                    arr(Bs), _ld(Bs[0]),
                                    float(beta), arr(C_locals), ldc, got, _stream(stream))
    _check(st, "tm_sgemm_dist_loopback")
    return [int(x) for x in got]


def summa_panels(k: int, pr: int, pc: int):
    """Panel plan of the 2-D SUMMA schedule: list of (k0, kr)."""
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.tm_summa_panel(k, pr, pc, -1, ctypes.byref(a), ctypes.byref(b)), "tm_summa_panel")
    out = []
    for i in range(a.value):
        _check(lib.tm_summa_panel(k, pr, pc, i, ctypes.byref(a), ctypes.byref(b)), "tm_summa_panel")
        out.append((a.value, b.value))
    return out


def summa_blocks(m, n, k, pr, pc, rank):
    """(rows_i, cols_j, ka_j, kb_i) of grid rank r = (r // pc, r % pc): each a
    (start, length) pair -- the blocks of C, A and B it owns (tm.h SUMMA)."""
    i, j = rank // pc, rank % pc
    return dist_rows(m, pr, i), dist_rows(n, pc, j), dist_rows(k, pc, j), dist_rows(k, pr, i)


def sgemm_summa_loopback(pr, pc, m, n, k, A_locals, B_locals, C_locals, alpha=1.0, beta=0.0, stream=None):
    """Single-process emulation of Comm.sgemm_summa over a pr x pc grid on the
    current GPU; A_locals[r], B_locals[r], C_locals[r] are rank r's blocks
    (summa_blocks).  Returns the panel bytes each simulated rank received."""
    P = pr * pc
    ptrs = lambda ts: (ctypes.c_void_p * P)(*[t.data_ptr() for t in ts])
    lds = lambda ts: (ctypes.c_int64 * P)(*[_ld(t) if t.shape[0] > 0 and t.shape[1] > 0 else max(1, t.shape[1]) for t in ts])
    got = (ctypes.c_uint64 * P)()
    st = lib.tm_sgemm_summa_loopback(pr, pc, m, n, k, float(alpha), ptrs(A_locals), lds(A_locals), ptrs(B_locals),
                                     lds(B_locals), float(beta), ptrs(C_locals), lds(C_locals), got, _stream(stream))
    _check(st, "tm_sgemm_summa_loopback")
    return [int(x) for x in got]


def _image(name, t, rows=None, cols=None):
    """(pointer, row pitch in floats) of an (N, M, 3) float32 CUDA image whose
    rows may be padded (strides (ld, 3, 1))."""
    _f32(name, t)
    if t.dim() != 3 or t.shape[2] != 3:
        raise ValueError(f"{name} must have shape (N, M, 3), got {tuple(t.shape)}")
    if rows is not None and tuple(t.shape[:2]) != (rows, cols):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected ({rows}, {cols}, 3)")
    if t.shape[1] > 0 and (t.stride(2) != 1 or (t.shape[1] > 1 and t.stride(1) != 3)):
        raise ValueError(f"{name}: each row must be 3*M contiguous floats")
    ld = int(t.stride(0)) if t.shape[0] > 1 else 3 * int(t.shape[1])
    return t.data_ptr(), ld


def blur(inp, out=None, stream=None):
    """The paper's two-stage 3x3 blur: inp (N, M, 3) ->
    out (N-2, M-2, 3), float32 CUDA tensors (rows may be padded)."""
    import torch
    N, M = int(inp.shape[0]), int(inp.shape[1])
    if out is None:
        out = torch.empty((N - 2, M - 2, 3), dtype=torch.float32, device=inp.device)
    _on_device(inp=inp, out=out)
    pi, ldi = _image("inp", inp)
    po, ldo = _image("out", out, N - 2, M - 2)
    _check(lib.tm_blur(N, M, pi, ldi, po, ldo, _stream(stream)), "tm_blur")
    return out


def blur_dist_loopback(N, M, lins, louts, stream=None):
    """Single-process emulation of Comm.blur over len(lins) simulated ranks:
    lins[r] (rows_r + 2, M, 3), louts[r] (rows_r, M-2, 3) with rows_r from
    dist_rows(N-2, P, r).  Returns the bytes each simulated rank received."""
    P = len(lins)
    infos_i = [_image("lin", t, dist_rows(N - 2, P, r)[1] + 2, M) for r, t in enumerate(lins)]
    infos_o = [_image("lout", t, dist_rows(N - 2, P, r)[1], M - 2) for r, t in enumerate(louts)]
    if len({ld for _, ld in infos_i}) != 1 or len({ld for _, ld in infos_o}) != 1:
        raise ValueError("every rank's lin (lout) must have the same row pitch")
    arr = lambda xs: (ctypes.c_void_p * P)(*[p for p, _ in xs])
    got = (ctypes.c_uint64 * P)()
    st = lib.tm_blur_dist_loopback(P, N, M, arr(infos_i), infos_i[0][1], arr(infos_o), infos_o[0][1], got,
                                   _stream(stream))
    _check(st, "tm_blur_dist_loopback")
    return [int(x) for x in got]


class IpcBuf(ctypes.Structure):
    """tm_ipc_buf: CUDA IPC handle of an allocation + byte offset (tm.h)."""
    _fields_ = [("bytes", ctypes.c_ubyte * 64), ("offset", ctypes.c_int64)]


def ipc_export(t) -> bytes:
    """72 bytes (tm_ipc_buf) naming the device buffer of tensor t for other processes."""
    b = IpcBuf()
    _check(lib.tm_ipc_export(ctypes.c_void_p(t.data_ptr()), ctypes.byref(b)), "tm_ipc_export")
    return ctypes.string_at(ctypes.addressof(b), ctypes.sizeof(b))


def _ipc_array(blobs):
    arr = (IpcBuf * len(blobs))()
    for i, blob in enumerate(blobs):
        ctypes.memmove(ctypes.addressof(arr[i]), blob, ctypes.sizeof(IpcBuf))
    return arr


class CeComm:
    """Copy-engine chain endpoint (tm_ce_*): B broadcast by copy engines over
    CUDA IPC mappings, no NCCL and no SMs taken from the GEMM.  Bootstrap and
    buffer-handle exchange go through a torch.distributed group (any backend)."""

    def __init__(self, rank: int, nranks: int, group=None):
        import torch.distributed as dist
        self.rank, self.nranks, self.group = rank, nranks, group
        h, fl = ctypes.c_void_p(), IpcBuf()
        _check(lib.tm_ce_create(ctypes.byref(h), nranks, rank, ctypes.byref(fl)), "tm_ce_create")
        self.handle = h
        blobs = [ctypes.string_at(ctypes.addressof(fl), ctypes.sizeof(fl))]
        if nranks > 1:
            allb = [None] * nranks
            dist.all_gather_object(allb, blobs[0], group=group)
            blobs = allb
        self._flags = _ipc_array(blobs)
        _check(lib.tm_ce_connect(self.handle, self._flags), "tm_ce_connect")

    def exchange(self, B):
        """All ranks' tm_ipc_export of their B buffers (collective): pass to sgemm
        as `handles`; valid while every rank keeps the same buffer."""
        import torch.distributed as dist
        mine = ipc_export(B)
        if self.nranks == 1:
            return _ipc_array([mine])
        allb = [None] * self.nranks
        dist.all_gather_object(allb, mine, group=self.group)
        return _ipc_array(allb)

    def sgemm(self, m, n, k, A_local, B, C_local, alpha=1.0, beta=0.0, root=0, stream=None, fused=False,
              handles=None):
        """Row-sharded C_local <- alpha*A_local@B + beta*C_local, B chain-broadcast
        from root by copy engines (tm_sgemm_dist_ce).  B: a dense k*ldb buffer on
        every rank.  handles: from exchange(B) (done here when None)."""
        if handles is None:
            handles = self.exchange(B)
        st = lib.tm_sgemm_dist_ce(self.handle, m, n, k, float(alpha), _ptr(A_local),
                                  _ld(A_local) if A_local is not None and A_local.shape[0] > 0 else max(k, 1),
                                  _ptr(B), _ld(B), handles, int(root), float(beta), _ptr(C_local),
                                  _ld(C_local) if C_local.shape[0] > 0 else max(n, 1), int(bool(fused)),
                                  _stream(stream))
        _check(st, "tm_sgemm_dist_ce")
        return C_local

    def bytes_received(self) -> int:
        v = ctypes.c_uint64()
        _check(lib.tm_ce_bytes_received(self.handle, ctypes.byref(v)), "tm_ce_bytes_received")
        return int(v.value)

    def close(self):
        if self.handle:
            _check(lib.tm_ce_destroy(self.handle), "tm_ce_destroy")
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def unique_id() -> bytes:
    """A fresh NCCL unique id (host-only)."""
    uid = (ctypes.c_ubyte * 128)()
    _check(lib.tm_comm_get_unique_id(ctypes.byref(uid)), "tm_comm_get_unique_id")
    return bytes(uid)


class Comm:
    """NCCL communicator owned by libtm (one process per GPU).

    Bootstrap: rank 0 creates the unique id, every rank receives it through the
    given torch.distributed process group (any backend), then all ranks init.
    """

    def __init__(self, rank: int, nranks: int, group=None):
        import torch
        import torch.distributed as dist
        uid = (ctypes.c_ubyte * 128)()
        if rank == 0:
            _check(lib.tm_comm_get_unique_id(ctypes.byref(uid)), "tm_comm_get_unique_id")
        if nranks > 1:
            obj = [bytes(uid) if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            ctypes.memmove(uid, obj[0], 128)
        h = ctypes.c_void_p()
        _check(lib.tm_comm_init(ctypes.byref(h), nranks, rank, ctypes.byref(uid)), "tm_comm_init")
        self.handle = h
        self.rank, self.nranks = rank, nranks
        self._torch = torch

    def close(self):
        if self.handle:
            _check(lib.tm_comm_destroy(self.handle), "tm_comm_destroy")
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, abort_on_error: bool = False) -> bool:
        """True if no asynchronous NCCL error was reported (failure detection)."""
        return lib.tm_comm_check(self.handle, int(abort_on_error)) == 0

    def bytes_received(self) -> int:
        v = ctypes.c_uint64()
        _check(lib.tm_comm_bytes_received(self.handle, ctypes.byref(v)), "tm_comm_bytes_received")
        return int(v.value)

    def sgemm(self, m, n, k, A_local, B, C_local, alpha=1.0, beta=0.0, root=0, stream=None, fused=False):
        """Row-sharded C_local <- alpha*A_local@B + beta*C_local; B broadcast from root.

        fused=False: K-chunked schedule (one GEMM per chunk, beta chain);
        fused=True: one flag-gated GEMM over the full K (tm_sgemm_dist_fused).
        Whole rows of B (ldb floats, padding included) are broadcast: B must be a
        k*ldb buffer on every rank (tm.h); use a dense B (ldb == n) for views."""
        fn = lib.tm_sgemm_dist_fused if fused else lib.tm_sgemm_dist
        st = fn(self.handle, m, n, k, float(alpha), _ptr(A_local),
                _ld(A_local) if A_local is not None and A_local.shape[0] > 0 else max(k, 1),
                _ptr(B), _ld(B), int(root), float(beta), _ptr(C_local),
                _ld(C_local) if C_local.shape[0] > 0 else max(n, 1), _stream(stream))
        _check(st, "tm_sgemm_dist_fused" if fused else "tm_sgemm_dist")
        return C_local

    def sgemm_allgather(self, m, n, k, A_local, B_shard, B_full, C_local, alpha=1.0, beta=0.0, stream=None):
        """B_shard (k/P x n) of every rank all-gathered into B_full (k x n), then the
        row-sharded GEMM.  Whole rows (ldb floats) move: B_shard must span
        (k/P)*ldb floats and B_full k*ldb (tm.h); use dense tensors for views."""
        st = lib.tm_sgemm_dist_allgather(self.handle, m, n, k, float(alpha), _ptr(A_local),
                                         _ld(A_local) if A_local.shape[0] > 0 else max(k, 1), _ptr(B_shard),
                                         _ptr(B_full), _ld(B_full), float(beta), _ptr(C_local),
                                         _ld(C_local) if C_local.shape[0] > 0 else max(n, 1), _stream(stream))
        _check(st, "tm_sgemm_dist_allgather")
        return C_local

    def blur(self, N, M, lin, lout, stream=None):
        """Row-distributed blur: lin (rows + 2, M, 3) holds
        this rank's input rows plus the 2-row border region (received from rank
        r+1; the last rank supplies input rows N-2, N-1 there), lout (rows, M-2, 3);
        rows from dist_rows(N-2, P, rank)."""
        rows = dist_rows(N - 2, self.nranks, self.rank)[1]
        pi, ldi = _image("lin", lin, rows + 2, M)
        po, ldo = _image("lout", lout, rows, M - 2)
        _check(lib.tm_blur_dist(self.handle, N, M, pi, ldi, po, ldo, _stream(stream)), "tm_blur_dist")
        return lout

    def sgemm_summa(self, pr, pc, m, n, k, A_local, B_local, C_local, alpha=1.0, beta=0.0, stream=None):
        """2-D SUMMA over a pr x pc grid (tm_sgemm_summa): this rank's blocks
        (summa_blocks(m, n, k, pr, pc, rank)); C_local updated in place."""
        ld = lambda t, w: _ld(t) if t is not None and t.shape[0] > 0 and t.shape[1] > 0 else max(1, w)
        st = lib.tm_sgemm_summa(self.handle, int(pr), int(pc), m, n, k, float(alpha), _ptr(A_local),
                                ld(A_local, A_local.shape[1]), _ptr(B_local), ld(B_local, B_local.shape[1]),
                                float(beta), _ptr(C_local), ld(C_local, C_local.shape[1]), _stream(stream))
        _check(st, "tm_sgemm_summa")
        return C_local

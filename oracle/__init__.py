"""CPU oracle for the tm_sgemm hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` leg may import this package.  The product package
(``paper_1804_10694_b200``) never imports it and shares no code with it.

The arithmetic lives in ``oracle/oracle.c`` (plain C, fp64, see its header for
the definition it writes out, PAPER.md:67 ``C = alpha*A*B + beta*C``).  This
module only compiles it (gcc, portable flags) and marshals numpy arrays.

Pinned by ``tests/test_oracle.py`` (exact rationals, numpy float64 matmul,
closed forms, integer inputs, golden example).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

# Portable flags: the .so built here also runs on the GPU box's host CPU.
# -ffp-contract=off keeps every fp64 operation a separately rounded op.
CFLAGS = ["-O3", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (no-op when up to date)."""
    if os.environ.get("TM_ORACLE_LIB"):
        return os.environ["TM_ORACLE_LIB"]
    import hashlib
    with _lock:
        with open(_SRC, "rb") as f:
            digest = hashlib.sha256(f.read() + " ".join(CFLAGS).encode()).hexdigest()
        stamp = _LIB + ".build.json"
        try:
            with open(stamp) as f:
                stale = not os.path.exists(_LIB) or f.read().strip() != digest
        except OSError:
            stale = True
        if force or stale:
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
            os.replace(tmp, _LIB)
            with open(stamp, "w") as f:
                f.write(digest)
    return _LIB


def build_mutant(n: int, out: str) -> str:
    """Compile oracle.c with -DORACLE_MUTANT=n (one step broken on purpose, see
    oracle.c) into ``out``; used only by tests/test_oracle_mutants.py, which
    loads it through TM_ORACLE_LIB in a subprocess and expects the pins to fail."""
    subprocess.check_call(["gcc", *CFLAGS, f"-DORACLE_MUTANT={int(n)}", _SRC, "-o", out, "-lm"])
    return out


def _load():
    global _lib
    if _lib is None:
        path = build()
        lib = ctypes.CDLL(path)
        i64, f32, vp = ctypes.c_int64, ctypes.c_float, ctypes.c_void_p
        lib.tm_oracle_sgemm_rows.argtypes = [i64, i64, i64, f32, vp, i64, vp, i64,
                                             f32, vp, i64, i64, vp, vp, vp, i64]
        lib.tm_oracle_sgemm_rows.restype = ctypes.c_int
        lib.tm_oracle_sgemm_op_rows.argtypes = [ctypes.c_int, ctypes.c_int, i64, i64, i64, f32, vp, i64, vp, i64,
                                                f32, vp, i64, i64, vp, vp, vp, i64]
        lib.tm_oracle_sgemm_op_rows.restype = ctypes.c_int
        lib.tm_oracle_conv2d_nhwc.argtypes = [i64] * 8 + [f32, vp, vp, f32, vp, i64, vp, vp, vp]
        lib.tm_oracle_conv2d_nhwc.restype = ctypes.c_int
        lib.tm_oracle_sgemm_f64.argtypes = [i64, i64, i64, f32, vp, i64, vp, i64,
                                            f32, vp, i64, vp, vp, i64]
        lib.tm_oracle_sgemm_f64.restype = ctypes.c_int
        lib.tm_oracle_dist_rows.argtypes = [i64, ctypes.c_int, ctypes.c_int,
                                            ctypes.POINTER(i64), ctypes.POINTER(i64)]
        lib.tm_oracle_dist_rows.restype = ctypes.c_int
        lib.tm_oracle_blur.argtypes = [i64, i64, vp, i64, vp, vp, vp]
        lib.tm_oracle_blur.restype = ctypes.c_int
        lib.tm_oracle_set_threads.argtypes = [ctypes.c_int]
        lib.tm_oracle_get_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def _check_f32(name, a):
    if a is None:
        return None
    if not isinstance(a, np.ndarray) or a.dtype != np.float32:
        raise TypeError(f"{name} must be a float32 numpy array")
    if a.ndim != 2 or (a.size > 0 and a.shape[1] > 1 and a.strides[1] != 4):
        raise ValueError(f"{name} must be 2-D with unit column stride")
    return a


def _ld(a):
    if a.shape[0] > 1 and a.size > 0:
        return a.strides[0] // 4
    return max(a.shape[1], 1)


def sgemm(alpha, A, B, beta, C0, rows=None, m=None, n=None, k=None, opa="N", opb="N"):
    """R, D for ``C = alpha*op(A)@op(B) + beta*C0`` (fp64), optionally only ``rows``.

    op(X) = X for "N", X.T for "T" (as stored: A is m x k for "N", k x m for
    "T"; B is k x n for "N", n x k for "T").  Float32 row-major views with any
    leading dimension.  A/B may be None when alpha == 0 or k == 0, C0 may be
    None when beta == 0 (they are then not read, reading 5).  Returns (R, D) as
    float64 arrays of shape (len(rows) or m, n).
    """
    A = _check_f32("A", A)
    B = _check_f32("B", B)
    C0 = _check_f32("C0", C0)
    ta, tb = int(opa == "T"), int(opb == "T")
    if m is None:
        m = (A.shape[1] if ta else A.shape[0]) if A is not None else C0.shape[0]
    if k is None:
        k = (A.shape[0] if ta else A.shape[1]) if A is not None else (
            (B.shape[1] if tb else B.shape[0]) if B is not None else 0)
    if n is None:
        n = (B.shape[0] if tb else B.shape[1]) if B is not None else C0.shape[1]
    lda = _ld(A) if A is not None else max(m if ta else k, 1)
    ldb = _ld(B) if B is not None else max(k if tb else n, 1)
    ldc = _ld(C0) if C0 is not None else max(n, 1)
    if rows is None:
        nrows, rows_arr = m, None
    else:
        rows_arr = np.ascontiguousarray(rows, dtype=np.int64)
        nrows = rows_arr.shape[0]
    R = np.empty((nrows, n), dtype=np.float64)
    D = np.empty((nrows, n), dtype=np.float64)
    rc = _load().tm_oracle_sgemm_op_rows(ta, tb, m, n, k, float(alpha), _ptr(A), lda, _ptr(B), ldb,
                                         float(beta), _ptr(C0), ldc, nrows, _ptr(rows_arr),
                                         _ptr(R), _ptr(D), max(n, 1))
    if rc != 0:
        raise ValueError(f"tm_oracle_sgemm_rows rejected its arguments (rc={rc})")
    return R, D


def conv2d_nhwc(alpha, X, Wt, beta, Y0, pad, pixels=None):
    """R, D (fp64, shape (npix, F)) for the NHWC / KRSC stride-1 convolution
    Y = alpha * conv(X, Wt) + beta * Y0 (oracle.c: tm_oracle_conv2d_nhwc).
    X: (Nb, H, W, C) float32, Wt: (F, R, S, C) float32, Y0: (Nb, Ho, Wo, F) or None."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    Wt = np.ascontiguousarray(Wt, dtype=np.float32)
    Nb, H, W, C = X.shape
    F, R, S, C2 = Wt.shape
    assert C == C2
    Ho, Wo = H + 2 * pad - R + 1, W + 2 * pad - S + 1
    Y0c = None if Y0 is None else np.ascontiguousarray(Y0, dtype=np.float32)
    if pixels is None:
        npix, pix = Nb * Ho * Wo, None
    else:
        pix = np.ascontiguousarray(pixels, dtype=np.int64)
        npix = pix.shape[0]
    Rr = np.empty((npix, F), np.float64)
    Dd = np.empty((npix, F), np.float64)
    rc = _load().tm_oracle_conv2d_nhwc(Nb, H, W, C, F, R, S, pad, float(alpha), _ptr(X), _ptr(Wt), float(beta),
                                       _ptr(Y0c), npix, _ptr(pix), _ptr(Rr), _ptr(Dd))
    if rc != 0:
        raise ValueError(f"tm_oracle_conv2d_nhwc rejected its arguments (rc={rc})")
    return Rr, Dd


def blur(img, rows=None):
    """R, D (fp64, shape (len(rows) or N-2, M-2, 3)) of the paper's two-stage
    blur of an N x M x 3 float32 image (oracle.c tm_oracle_blur)."""
    img = np.ascontiguousarray(img, dtype=np.float32)
    N, M, C = img.shape
    assert C == 3
    if rows is None:
        nrows, r = N - 2, None
    else:
        r = np.ascontiguousarray(rows, dtype=np.int64)
        nrows = r.shape[0]
    R = np.empty((nrows, M - 2, 3), np.float64)
    D = np.empty((nrows, M - 2, 3), np.float64)
    if _load().tm_oracle_blur(N, M, _ptr(img), nrows, _ptr(r), _ptr(R), _ptr(D)) != 0:
        raise ValueError("tm_oracle_blur rejected its arguments")
    return R, D


def dist_rows(m, nranks, rank):
    """(row0, rows) of rank ``rank`` under the balanced row partition."""
    r0, nr = ctypes.c_int64(), ctypes.c_int64()
    if _load().tm_oracle_dist_rows(m, nranks, rank, ctypes.byref(r0), ctypes.byref(nr)) != 0:
        raise ValueError("invalid partition arguments")
    return r0.value, nr.value


def set_threads(n: int) -> None:
    _load().tm_oracle_set_threads(int(n))


def get_threads() -> int:
    return int(_load().tm_oracle_get_threads())


def normalized_error(C, R, D):
    """err[i,j] = |C - R| / D (north_star acceptance metric, computed in fp64).

    Where D == 0 the result must equal R exactly (reading 8): such elements
    report 0 if equal, +inf otherwise.
    """
    C = np.asarray(C, dtype=np.float64)
    diff = np.abs(C - R)
    with np.errstate(divide="ignore", invalid="ignore"):
        err = np.where(D > 0, diff / np.where(D > 0, D, 1.0), np.where(diff == 0, 0.0, np.inf))
    err = np.where(np.isnan(C) & ~np.isnan(R), np.inf, err)
    return err

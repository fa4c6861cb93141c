"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/tm.h declares, validates arguments on the host before any CUDA
call, dispatches paths by alignment, and has no CPU fallback."""
import ctypes
import os
import re

import pytest

import paper_1804_10694_b200 as tm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "tm.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tm_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    declared = _declared_symbols()
    assert len(declared) >= 15
    assert sorted(tm.EXPORTED_SYMBOLS) == declared
    L = ctypes.CDLL(tm.lib_path)
    for name in declared:
        assert getattr(L, name) is not None, name


def test_library_is_sm100a_only():
    """The .so carries only sm_100a SASS (no PTX for JIT, no other arch)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", tm.lib_path], capture_output=True,
                         text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_status_strings_and_version():
    assert tm.status_string(0) == "TM_OK"
    assert tm.status_string(1) == "TM_ERR_INVALID_VALUE"
    assert tm.status_string(2) == "TM_ERR_UNSUPPORTED_DEVICE"
    assert tm.lib.tm_get_version() >= 100


def _ex(m, n, k, alpha=1.0, A=16, lda=None, B=16, ldb=None, beta=0.0, C=1 << 20, ldc=None, algo=0):
    lda = max(k, 1) if lda is None else lda
    ldb = max(n, 1) if ldb is None else ldb
    ldc = max(n, 1) if ldc is None else ldc
    return tm.lib.tm_sgemm_ex(m, n, k, alpha, ctypes.c_void_p(A), lda, ctypes.c_void_p(B), ldb, beta,
                              ctypes.c_void_p(C), ldc, None, algo)


@pytest.mark.parametrize("args", [
    dict(m=-1, n=4, k=4),
    dict(m=4, n=-1, k=4),
    dict(m=4, n=4, k=-1),
    dict(m=4, n=4, k=8, lda=7),          # lda < k
    dict(m=4, n=8, k=4, ldb=7),          # ldb < n
    dict(m=4, n=8, k=4, ldc=7),          # ldc < n
    dict(m=4, n=4, k=4, A=0),            # NULL A while alpha != 0
    dict(m=4, n=4, k=4, B=0),            # NULL B
    dict(m=4, n=4, k=4, C=0),            # NULL C
    dict(m=4, n=4, k=4, A=1 << 20),      # C overlaps A
    dict(m=4, n=4, k=4, algo=9),         # unknown algo
    dict(m=4, n=4, k=4, C=(1 << 20) + 4, algo=1),  # TF32X3 forced on misaligned C
])
def test_invalid_arguments_rejected_on_host(args):
    assert _ex(**args) == 1  # TM_ERR_INVALID_VALUE, before any CUDA call


def test_noop_needs_no_device():
    assert _ex(0, 5, 5) == 0
    assert _ex(5, 0, 5) == 0


def test_no_cpu_fallback():
    """Valid arguments on a machine without a usable sm_100 device must fail,
    never silently compute on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert _ex(8, 8, 8) in (2, 3)  # UNSUPPORTED_DEVICE or CUDA error


def test_plan_dispatch_by_alignment():
    # aligned pointers + ld % 4 == 0 -> tensor cores; otherwise SIMT (never an error under AUTO)
    # small problems (m*n*k <= 2^22, k <= 256) take the latency-bound small kernel, aligned or not
    assert tm.plan_name(64, 64, 64, 1.0, 0.0, 1 << 12, 64, 1 << 16, 64, 1 << 24, 64) == "simt_small"
    assert tm.plan_name(64, 64, 64, 1.0, 0.0, (1 << 12) + 4, 64, 1 << 16, 64, 1 << 24, 64) == "simt_small"
    assert tm.plan_name(128, 128, 256, 1.0, 0.0, 1 << 12, 256, 1 << 16, 128, 1 << 28, 128) == "simt_small"
    assert tm.plan_name(64, 64, 260, 1.0, 0.0, 1 << 12, 260, 1 << 16, 64, 1 << 28, 64) == "tf32x3"  # deep K
    assert tm.plan_name(256, 256, 260, 1.0, 0.0, 1 << 12, 260, 1 << 16, 256, 1 << 28, 256) == "tf32x3"
    assert tm.plan_name(256, 255, 260, 1.0, 0.0, 1 << 12, 260, 1 << 16, 255, 1 << 28, 255) == "simt"
    assert tm.plan_name(512, 64, 1024, 1.0, 0.0, (1 << 12) + 4, 1024, 1 << 16, 64, 1 << 28, 64) == "simt"
    assert tm.plan_name(64, 64, 64, 1.0, 0.0, 1 << 12, 64, 1 << 16, 64, 1 << 24, 64, algo=2) == "simt"
    assert tm.plan_name(64, 64, 64, 1.0, 0.0, 1 << 12, 64, 1 << 16, 64, 1 << 24, 64, algo=3) == "tf32x1"
    # special cases
    assert tm.plan_name(64, 64, 64, 0.0, 0.5, 0, 64, 0, 64, 1 << 24, 64) == "scale"
    assert tm.plan_name(64, 64, 0, 1.0, 0.5, 0, 1, 0, 64, 1 << 24, 64) == "scale"
    assert tm.plan_name(0, 64, 64, 1.0, 0.5, 0, 64, 0, 64, 0, 64) == "noop"
    assert tm.plan_name(-1, 64, 64) == "invalid"


def test_dist_rows_partition():
    for m in [0, 1, 5, 1060, 16384, 16387]:
        for P in [1, 2, 3, 4, 8]:
            seen = []
            for r in range(P):
                r0, nr = tm.dist_rows(m, P, r)
                seen.extend(range(r0, r0 + nr))
            assert seen == list(range(m))
    # the product's partition is the oracle's (pinned by tests/golden/dist_rows.json)
    import oracle
    for m in list(range(0, 40)) + [1060, 16383, 16384, 16387]:
        for P in range(1, 10):
            for r in range(P):
                assert tm.dist_rows(m, P, r) == oracle.dist_rows(m, P, r), (m, P, r)
    with pytest.raises(tm.TmError):
        tm.dist_rows(10, 0, 0)
    with pytest.raises(tm.TmError):
        tm.dist_rows(10, 2, 2)


def test_product_package_never_imports_oracle():
    """The product path shares no code with the oracle."""
    pkg = os.path.join(ROOT, "paper_1804_10694_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                with open(os.path.join(dirpath, f)) as fh:
                    src = fh.read()
                assert "oracle" not in src.replace("# no oracle", ""), f


def test_op_and_colmajor_validation_on_host():
    L = tm.lib
    vp = ctypes.c_void_p
    # opa = T: lda must be >= m
    assert L.tm_sgemm_op(1, 0, 64, 8, 16, 1.0, vp(16), 32, vp(1 << 16), 8, 0.0, vp(1 << 24), 8, None, 0) == 1
    # opb = T: ldb must be >= k
    assert L.tm_sgemm_op(0, 1, 8, 64, 16, 1.0, vp(16), 16, vp(1 << 16), 8, 0.0, vp(1 << 24), 64, None, 0) == 1
    assert L.tm_sgemm_op(2, 0, 8, 8, 8, 1.0, vp(16), 8, vp(1 << 16), 8, 0.0, vp(1 << 24), 8, None, 0) == 1
    # explicit tensor-core paths (3xTF32, 1xTF32) reject a misaligned operand
    assert L.tm_sgemm_op(1, 0, 8, 8, 8, 1.0, vp(20), 8, vp(1 << 16), 8, 0.0, vp(1 << 24), 8, None, 3) == 1
    assert L.tm_sgemm_op(0, 1, 8, 8, 8, 1.0, vp(16), 8, vp(1 << 16), 10, 0.0, vp(1 << 24), 8, None, 1) == 1
    assert L.tm_sgemm_colmajor(b"X", b"N", 8, 8, 8, 1.0, vp(16), 8, vp(1 << 16), 8, 0.0, vp(1 << 24), 8, None) == 1
    assert L.tm_sgemm_op(1, 1, 0, 8, 8, 1.0, vp(16), 8, vp(1 << 16), 8, 0.0, vp(1 << 24), 8, None, 0) == 0  # noop


def test_binding_rejects_mismatched_shapes_and_host_tensors():
    """The binding checks shapes (as torch.mm does) and devices before any
    pointer reaches a kernel (ValueError, nothing launched)."""
    import numpy as np
    import torch
    A, B, C = torch.zeros(8, 4), torch.zeros(4, 6), torch.zeros(8, 6)
    with pytest.raises(ValueError):
        tm.sgemm(torch.zeros(7, 4), B, C)          # A has fewer than m rows
    with pytest.raises(ValueError):
        tm.sgemm(A, torch.zeros(3, 6), C)          # B has fewer than k rows
    with pytest.raises(ValueError):
        tm.sgemm_op(A, torch.zeros(6, 5), C, opb="T")
    with pytest.raises(ValueError):
        tm.sgemm(A, B, C)                          # host tensors are not device tensors
    with pytest.raises(ValueError):
        tm.sgemm_host(A.numpy(), B.numpy()[:, ::2].copy()[:, :3], C.numpy())  # shape mismatch
    Bs = np.zeros((4, 12), np.float32)[:, ::2]     # non-unit column stride
    with pytest.raises(ValueError):
        tm.sgemm_host(A.numpy(), Bs, C.numpy())
    with pytest.raises(ValueError):
        tm.sgemm_host(A.numpy(), np.zeros((4, 6), np.float32)[::-1], C.numpy())  # negative row stride


@pytest.mark.parametrize("args", [
    dict(N=2, M=5),                      # fewer than 3 rows: no output of the 3x3 stencil
    dict(N=5, M=2),                      # fewer than 3 columns
    dict(N=5, M=5, ldi=14),              # ldi < 3M
    dict(N=5, M=5, ldo=8),               # ldo < 3(M-2)
    dict(N=5, M=5, inp=0),               # NULL in
    dict(N=5, M=5, out=0),               # NULL out
    dict(N=5, M=5, out=(1 << 20) + 40),  # out overlaps in
])
def test_blur_invalid_arguments_rejected_on_host(args):
    N, M = args["N"], args["M"]
    st = tm.lib.tm_blur(N, M, ctypes.c_void_p(args.get("inp", 1 << 20)), args.get("ldi", 3 * M),
                        ctypes.c_void_p(args.get("out", 1 << 24)), args.get("ldo", 3 * max(M - 2, 1)), None)
    assert st == 1


def test_blur_dist_loopback_rejects_bad_rank_count_on_host():
    P = (ctypes.c_void_p * 1)(1 << 20)
    assert tm.lib.tm_blur_dist_loopback(0, 9, 9, P, 27, P, 21, None, None) == 1


def test_conv_plan_names_for_the_paper_filter_sizes():
    """PAPER.md:834-835 (3x3 ... 11x11 on 32x512x512x16, 16 filters): the direct
    kernel takes all of them (9x9 in passes of filter rows; 11x11, whose
    resident filters would need 2 x 11 x 176 x 64 B, in two launches over the
    filter columns); 25x25 does not fit a warp's shift -> implicit GEMM;
    channels not a multiple of 16 -> SIMT; host-only."""
    assert tm.conv2d_plan_name(1, 64, 64, 16, 16, 25, 25, 12) == "implicit_gemm"
    for r, want in ((1, "direct"), (3, "direct"), (5, "direct"), (7, "direct"), (9, "direct"), (11, "direct_split")):
        assert tm.conv2d_plan_name(32, 512, 512, 16, 16, r, r, r // 2) == want, r
    assert tm.conv2d_plan_name(1, 8, 8, 18, 16, 3, 3, 1) == "simt"
    assert tm.conv2d_plan_name(1, 8, 8, 16, 16, 3, 3, 1, alpha=0.0) == "scale"
    assert tm.conv2d_plan_name(1, 2, 2, 16, 16, 3, 3, 0) == "invalid"  # no output pixel


def _sk_ranges(iters, clusters):
    return [(iters * c // clusters, iters * (c + 1) // clusters) for c in range(clusters)]


def test_streamk_region_invariants():
    """Host-only stream-K split (tm_sgemm_streamk_region, the rule the kernel
    launch uses): every cluster owns at least two iterations of the region (an
    empty range would never publish the partial its tile's finalizer waits
    for), the tiles after the region form whole waves, and the modes select
    what DESIGN 6.1 says."""

    for clusters in (1, 2, 37, 74, 148):
        for tiles in (1, 2, 3, 36, 45, 73, 74, 75, 80, 100, 147, 148, 149, 196, 256, 300, 1025):
            for kb in (1, 2, 3, 18, 34, 63, 64, 128, 512):
                for mode in (-1, 0, 1, 2):
                    sk, cu = tm.streamk_region(tiles, kb, clusters, mode)
                    assert 0 <= sk <= tiles and 1 <= cu <= clusters, (tiles, kb, clusters, mode, sk, cu)
                    assert (tiles - sk) % cu == 0, (tiles, kb, clusters, mode, sk, cu)
                    iters = sk * kb
                    if sk < tiles:  # hybrid: every cluster keeps its full count
                        assert cu == clusters and iters >= 2 * cu
                    if iters >= 2:
                        assert all(e - b >= 2 for b, e in _sk_ranges(iters, cu)), (tiles, kb, clusters, mode, sk, cu)
                    if mode == 0:
                        assert sk == tiles
    # the cases of DESIGN 6.1: C3 (256 tiles of 128 K-blocks on 74 clusters) splits its
    # partial wave; C4 (196 of 18) the partial wave plus one wave; 80 tiles of 2
    # K-blocks (12 iterations for 74 clusters) falls back to pure stream-K on 80 clusters
    assert tm.streamk_region(256, 128, 74) == (34, 74)
    assert tm.streamk_region(196, 18, 74) == (48 + 74, 74)
    assert tm.streamk_region(80, 2, 74) == (80, 74)
    assert tm.streamk_region(30, 1, 74) == (30, 15)
    with pytest.raises(tm.TmError):
        tm.streamk_region(0, 1, 74)


def test_plan_config_large_shapes():
    """Host-only planner at BASELINE.json's sizes: the tensor-core path, the
    cluster tile and the schedule DESIGN 6.1 / BASELINE.md report (stream-K for
    the partial-wave shapes C2/C3/C4, data-parallel for C3b/C5)."""
    TC = 3
    assert tm.plan_config(16384, 16384, 16384, 1.5, 0.5) == (TC, 2, 128, 0)
    assert tm.plan_config(8192, 8192, 8192, 1.5, 0.5) == (TC, 2, 128, 0)
    assert tm.plan_config(4096, 4096, 4096, 1.5, 0.5) == (TC, 2, 128, 1)
    assert tm.plan_config(50176, 64, 576, 1.5, 0.5) == (TC, 2, 32, 1)
    assert tm.plan_config(1060, 1060, 1060, 1.5, 0.5) == (TC, 2, 64, 1)

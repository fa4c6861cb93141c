"""Hardware-semantics probes of kind::tf32 tcgen05.mma, run
through the single-pass TF32 path of the C ABI:

1. operand conversion: does the tensor core truncate the low 13 mantissa bits
   of a raw fp32 operand (the 3xTF32 design relies on it: the raw TMA tile is
   used as `hi`), or round it?
2. accumulation rounding: within one MMA (K=8) and across MMAs.

Results are written to gpurun_out/probes.json for DESIGN.md."""
import json
import os

import numpy as np
import pytest

from gpu_util import run

pytestmark = pytest.mark.gpu
TF32X1 = 3


def _bits(x):
    return np.asarray(x, dtype=np.float32).view(np.uint32)


def _from_bits(b):
    return np.asarray(b, dtype=np.uint32).view(np.float32)


def _record(key, value):
    os.makedirs("gpurun_out", exist_ok=True)
    path = "gpurun_out/probes.json"
    d = {}
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
    d[key] = value
    with open(path, "w") as f:
        json.dump(d, f, indent=1)


def _patterns(n):
    g = np.random.Generator(np.random.PCG64(5))
    base = _bits(g.uniform(0.5, 2.0, n).astype(np.float32)) & np.uint32(0xFFFFE000)
    low = np.array([0x0, 0x1, 0xFFF, 0x1000, 0x1001, 0x1FFF, 0x0800, 0x17FF], dtype=np.uint32)
    low = np.resize(low, n)
    sign = np.where(np.arange(n) % 2 == 0, 0, 0x80000000).astype(np.uint32)
    return _from_bits(base | low | sign)


def _classify(x, got):
    b = _bits(x)
    trunc = _from_bits(b & np.uint32(0xFFFFE000))
    mag = b & np.uint32(0x7FFFFFFF)
    low = mag & np.uint32(0x1FFF)
    up = _from_bits((b & np.uint32(0xFFFFE000)) + np.uint32(0x2000))
    rna = np.where(low >= 0x1000, up, trunc)
    odd = (mag >> np.uint32(13)) & np.uint32(1)
    rne = np.where((low > 0x1000) | ((low == 0x1000) & (odd == 1)), up, trunc)
    return {"trunc": bool(np.array_equal(got, trunc)), "rna": bool(np.array_equal(got, rna)),
            "rne": bool(np.array_equal(got, rne))}


def test_operand_conversion_A_and_B():
    n = 128
    x = _patterns(n)
    # A operand (K-major): A[:, 0] = x, B[0, 0] = 1  ->  C[:, 0] = cvt(x)
    A = np.zeros((n, 8), np.float32)
    A[:, 0] = x
    B = np.zeros((8, 16), np.float32)
    B[0, 0] = 1.0
    C, _ = run(A, B, np.zeros((n, 16), np.float32), 1.0, 0.0, TF32X1)
    ra = _classify(x, C[:, 0])
    # B operand (MN-major): B[0, :] = x, A[0, 0] = 1  ->  C[0, :] = cvt(x)
    A2 = np.zeros((16, 8), np.float32)
    A2[0, 0] = 1.0
    B2 = np.zeros((8, n), np.float32)
    B2[0, :] = x
    C2, _ = run(A2, B2, np.zeros((16, n), np.float32), 1.0, 0.0, TF32X1)
    rb = _classify(x, C2[0, :])
    _record("operand_A", ra)
    _record("operand_B", rb)
    assert any(ra.values()) and any(rb.values()), (ra, rb)
    # The 3xTF32 split (hi = raw operand) is only exact if the hardware truncates.
    assert ra["trunc"] and rb["trunc"], (ra, rb)


def test_accumulation_rounding():
    """1 + 0.75 ulp(1): RN gives 1 + ulp, RZ gives 1.  Within one MMA (both
    products in one K=8 group) and across MMAs (second product at k = 8)."""
    ulp = 2.0 ** -23
    res = {}
    for where, kk in (("within_mma", 1), ("across_mma", 8), ("across_kblock", 32)):
        K = 40
        A = np.zeros((128, K), np.float32)
        A[:, 0] = 1.0
        A[:, kk] = np.float32(0.75 * ulp)
        B = np.zeros((K, 16), np.float32)
        B[:, 0] = 1.0
        C, _ = run(A, B, np.zeros((128, 16), np.float32), 1.0, 0.0, TF32X1)
        v = float(C[0, 0])
        res[where] = "RN" if v == 1.0 + ulp else ("RZ" if v == 1.0 else repr(v))
        # negative: -1 - 0.75ulp -> RN -1-ulp, RZ -1
        A[:, 0] = -1.0
        A[:, kk] = np.float32(-0.75 * ulp)
        C, _ = run(A, B, np.zeros((128, 16), np.float32), 1.0, 0.0, TF32X1)
        v = float(C[0, 0])
        res[where + "_neg"] = "RN" if v == -1.0 - ulp else ("RZ" if v == -1.0 else repr(v))
    _record("accumulation", res)
    assert all(r in ("RN", "RZ") for r in res.values()), res

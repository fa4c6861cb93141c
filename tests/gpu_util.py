"""Helpers for GPU parity tests: move seeded numpy inputs to the device with
chosen leading dimensions / guard bands, run a path through the C ABI, and
score the result against the oracle (tests only)."""
import os

import numpy as np

import oracle

SENTINEL = np.float32(-12345.5)


def to_dev(x, ld=None, guard_rows=0, fill=SENTINEL):
    """Device copy of 2-D float32 `x` inside a (rows+guard_rows) x ld buffer
    pre-filled with `fill`; returns (view, full_buffer)."""
    import torch
    r, c = x.shape
    ld = c if ld is None else ld
    buf = torch.full((r + guard_rows, max(ld, 1)), float(fill), dtype=torch.float32, device="cuda")
    if r and c:
        buf[:r, :c] = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return buf[:r, :c], buf


def run(A, B, C0, alpha, beta, algo, lda=None, ldb=None, ldc=None, guard_rows=0, config=None, c_fill=None):
    """Runs tm_sgemm_ex on device copies; returns (C_result numpy, C buffer numpy)."""
    import torch
    import paper_1804_10694_b200 as tm
    dA = to_dev(A, lda)[0] if A is not None else None
    dB = to_dev(B, ldb)[0] if B is not None else None
    dC, cbuf = to_dev(C0, ldc, guard_rows)
    if c_fill is not None:
        dC.fill_(c_fill)
    old = os.environ.get("TM_TC_CONFIG")
    if config:
        os.environ["TM_TC_CONFIG"] = config
    try:
        k = A.shape[1] if A is not None else 0
        tm.sgemm_ex(dA, dB, dC, alpha, beta, algo, m=C0.shape[0], n=C0.shape[1], k=k)
        torch.cuda.synchronize()
    finally:
        if config:
            if old is None:
                del os.environ["TM_TC_CONFIG"]
            else:
                os.environ["TM_TC_CONFIG"] = old
    return dC.cpu().numpy(), cbuf.cpu().numpy()


def max_err(C, A, B, C0, alpha, beta, rows=None):
    R, D = oracle.sgemm(alpha, A, B, beta, C0, rows=rows)
    Cs = C if rows is None else C[rows]
    return float(np.max(oracle.normalized_error(Cs, R, D))) if Cs.size else 0.0

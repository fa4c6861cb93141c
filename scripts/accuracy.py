"""Accuracy survey of the GPU paths against the oracle on sampled rows of the
large configs, for zero-mean (gating) and all-positive (stress) inputs.
Prints one JSON line per case."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_1804_10694_b200 as tm  # noqa: E402
import seeded_inputs as si  # noqa: E402

cases = sys.argv[1:] or ["C3b:uniform", "C3b:positive", "C5:uniform", "C5:positive"]
for case in cases:
    cfg, kind = case.split(":")
    algo = tm.ALGO_TF32X3
    m, n, k = si.CONFIGS[cfg]
    t0 = time.time()
    A, B, C0 = si.matrices(m, n, k, si.SEEDS[cfg], kind=kind)
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C0))
    tm.sgemm_ex(dA, dB, dC, si.ALPHA, si.BETA, algo)
    torch.cuda.synchronize()
    rows = si.sample_rows(m, count=48, tile=256)
    C = dC[torch.from_numpy(rows).cuda()].cpu().numpy()
    R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0, rows=rows)
    err = oracle.normalized_error(C, R, D)
    print(json.dumps({"case": case, "m": m, "n": n, "k": k, "rows": len(rows), "max_err": float(err.max()),
                      "p99_99": float(np.quantile(err, 0.9999)), "mean_err": float(err.mean()),
                      "secs": round(time.time() - t0, 1)}), flush=True)
    del dA, dB, dC
    torch.cuda.empty_cache()

"""Summarise TM_TRACE_PATH timelines: per slot, min/median/max over CTAs of
(t_slot - t_kernel_start_min) in microseconds."""
import json
import sys

import numpy as np

NAMES = ["entry", "setup_done", "producer_done", "partials_drained(last unit)", "first_mma", "last_mma_issued",
         "acc_done(last unit)", "epilogue_done(last unit)", "first_stage_landed", "partial_published",
         "finalizer_flag_acquired", "teardown_barrier"]
for line in open(sys.argv[1]):
    d = json.loads(line)
    t = np.array(d["t"], dtype=np.float64).reshape(d["ctas"], -1)
    t0 = t[:, 0][t[:, 0] > 0].min()
    print(f"cg={d['cg']} bn={d['bn']} sk={d['sk']} {d['m']}x{d['n']}x{d['k']} ctas={d['ctas']}")
    for i, nm in enumerate(NAMES):
        v = t[:, i]
        v = v[v > 0] - t0
        if len(v):
            print(f"   {nm:26s} min {v.min()/1e3:8.2f}  med {np.median(v)/1e3:8.2f}  max {v.max()/1e3:8.2f} us  (n={len(v)})")
    # per-CTA intervals (both marks present in the same CTA)
    pairs = [(1, 8, "setup -> first stage landed"), (8, 4, "first stage -> first MMA"), (4, 5, "first -> last MMA"),
             (5, 3, "last MMA -> last partial drained"), (3, 9, "drained -> partial published"),
             (3, 10, "drained -> finalizer flag acquired"), (3, 6, "drained -> acc done"),
             (6, 7, "acc done -> epilogue done"), (7, 11, "epilogue done -> teardown barrier")]
    for a, b, nm in pairs:
        if t.shape[1] <= max(a, b):
            continue
        ok = (t[:, a] > 0) & (t[:, b] > 0)
        if ok.any():
            dlt = (t[ok, b] - t[ok, a]) / 1e3
            print(f"   d[{nm:34s}] min {dlt.min():7.2f}  med {np.median(dlt):7.2f}  max {dlt.max():7.2f} us  (n={ok.sum()})")

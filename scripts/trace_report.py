"""Summarise TM_TRACE_PATH timelines: per slot, min/median/max over CTAs of
(t_slot - t_kernel_start_min) in microseconds."""
import json
import sys

import numpy as np

NAMES = ["entry", "setup_done", "producer_done", "partials_drained(last unit)", "first_mma", "last_mma_issued",
         "acc_done(last unit)", "epilogue_done(last unit)"]
for line in open(sys.argv[1]):
    d = json.loads(line)
    t = np.array(d["t"], dtype=np.float64).reshape(d["ctas"], 8)
    t0 = t[:, 0][t[:, 0] > 0].min()
    print(f"cg={d['cg']} bn={d['bn']} sk={d['sk']} {d['m']}x{d['n']}x{d['k']} ctas={d['ctas']}")
    for i, nm in enumerate(NAMES):
        v = t[:, i]
        v = v[v > 0] - t0
        if len(v):
            print(f"   {nm:26s} min {v.min()/1e3:8.2f}  med {np.median(v)/1e3:8.2f}  max {v.max()/1e3:8.2f} us  (n={len(v)})")

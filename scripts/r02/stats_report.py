"""TM_EXP_STATS timelines: per CTA, the summed wait cycles of trace slots 12-15
(producer empty_raw waits [3 producers summed], split full / empty_lo waits,
MMA ready waits) beside the kernel span (globaltimer, slots 0 and 11)."""
import json, sys
import numpy as np
for line in open(sys.argv[1]):
    d = json.loads(line)
    t = np.array(d["t"], dtype=np.float64).reshape(d["ctas"], -1)
    span_ns = np.median(t[:, 11] - t[:, 0])
    print(f"cg={d['cg']} bn={d['bn']} sk={d['sk']} {d['m']}x{d['n']}x{d['k']}: kernel span med {span_ns/1e3:.2f} us")
    for k, nm in ((12, "producers wait empty_raw (sum of 3)"), (13, "split wait full"), (14, "split wait empty_lo"),
                  (15, "MMA wait ready")):
        v = t[:, k][t[:, k] > 0]
        if len(v):
            print(f"   {nm:36s} med {np.median(v):10.0f} cyc  ({np.median(v)/1.9e3:.2f} us at 1.9 GHz)")

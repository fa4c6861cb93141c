"""Times every tensor-core configuration (cg, bn, stream-K) on a set of shapes in
one process (CUDA events, L2 flushed by a 512 MiB read between reps) and
prints the best per shape, plus what the planner picks.  Planner calibration
tool."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_10694_b200 as tm  # noqa: E402

SHAPES = [(1060, 1060, 1060), (2048, 2048, 2048), (3000, 3000, 3000), (4096, 4096, 4096), (50176, 64, 576),
          (8192, 8192, 1024), (1024, 8192, 8192), (8192, 1024, 8192), (16384, 128, 4096), (512, 512, 16384)]
if len(sys.argv) > 1:
    SHAPES = [tuple(int(x) for x in s.split("x")) for s in sys.argv[1:]]
CFGS = [f"{cg},{bn},{sk}" for cg in (2, 1) for bn in (128, 64, 32) for sk in (0, 1)]
flush = torch.ones(512 * 2 ** 20 // 4, device="cuda")
out = torch.empty(1, device="cuda")


def time_cfg(A, B, C, cfg, reps=10):
    if cfg:
        os.environ["TM_TC_CONFIG"] = cfg
    else:
        os.environ.pop("TM_TC_CONFIG", None)
    for _ in range(2):
        tm.sgemm(A, B, C, 1.5, 0.5)
    ts = []
    for _ in range(reps):
        torch.sum(flush, dim=0, out=out[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tm.sgemm(A, B, C, 1.5, 0.5)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


for (m, n, k) in SHAPES:
    A = torch.rand(m, k, device="cuda")
    B = torch.rand(k, n, device="cuda")
    C = torch.rand(m, n, device="cuda")
    res = {c: time_cfg(A, B, C, c) for c in CFGS}
    auto = time_cfg(A, B, C, None)
    best = min(res, key=res.get)
    fl = 2.0 * m * n * k
    print(json.dumps({"shape": f"{m}x{n}x{k}", "best": best, "best_ms": round(res[best], 4),
                      "best_tflops": round(fl / res[best] / 1e9, 1), "auto_ms": round(auto, 4),
                      "auto_vs_best": round(res[best] / auto, 3),
                      "all": {c: round(v, 4) for c, v in sorted(res.items(), key=lambda kv: kv[1])}}), flush=True)
    del A, B, C
    torch.cuda.empty_cache()

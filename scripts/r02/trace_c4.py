"""One traced C4 call (50176x64x576, beta 0.5, after an L2 flush) per TM_TC_CONFIG; TM_TRACE_PATH timeline."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1804_10694_b200 as tm
out = sys.argv[1]
m, n, k = 50176, 64, 576
flush = torch.ones(512 * 2 ** 20 // 4, device="cuda"); fo = torch.empty(1, device="cuda")
g = torch.Generator(device="cuda"); g.manual_seed(1)
A = torch.rand(m, k, device="cuda", generator=g); B = torch.rand(k, n, device="cuda", generator=g)
C = torch.rand(m, n, device="cuda", generator=g)
for cfg in sys.argv[2:]:
    if cfg != "auto":
        os.environ["TM_TC_CONFIG"] = cfg
    for _ in range(3):
        tm.sgemm_ex(A, B, C, 1.5, 0.5, 1)
    torch.sum(flush, dim=0, out=fo[0]); torch.cuda.synchronize()
    os.environ["TM_TRACE_PATH"] = out
    tm.sgemm_ex(A, B, C, 1.5, 0.5, 1)
    torch.cuda.synchronize()
    del os.environ["TM_TRACE_PATH"]
    os.environ.pop("TM_TC_CONFIG", None)

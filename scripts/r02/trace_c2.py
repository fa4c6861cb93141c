"""One traced C2 call (after an L2 flush) per (config, beta); TM_TRACE_PATH timeline."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1804_10694_b200 as tm
out = sys.argv[1]
s = int(os.environ.get("SIZE", "1060"))
flush = torch.ones(512 * 2 ** 20 // 4, device="cuda"); fo = torch.empty(1, device="cuda")
g = torch.Generator(device="cuda"); g.manual_seed(1)
A, B, C = (torch.rand(s, s, device="cuda", generator=g) for _ in range(3))
for cfg in sys.argv[2:]:
    c, beta = cfg.split("/")
    os.environ["TM_TC_CONFIG"] = c
    for _ in range(3):
        tm.sgemm_ex(A, B, C, 1.5, float(beta), 1)
    torch.sum(flush, dim=0, out=fo[0]); torch.cuda.synchronize()
    os.environ["TM_TRACE_PATH"] = out
    tm.sgemm_ex(A, B, C, 1.5, float(beta), 1)
    torch.cuda.synchronize()
    del os.environ["TM_TRACE_PATH"]

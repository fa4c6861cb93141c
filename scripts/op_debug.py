"""Run one sgemm_op case (argv: opa opb m n k [algo]) and sync -- for compute-sanitizer."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1804_10694_b200 as tm
opa, opb = sys.argv[1], sys.argv[2]
m, n, k = (int(x) for x in sys.argv[3:6])
algo = int(sys.argv[6]) if len(sys.argv) > 6 else 1
pad = lambda x: (x + 3) // 4 * 4
ar, ac = (k, m) if opa == "T" else (m, k)
br, bc = (n, k) if opb == "T" else (k, n)
A = torch.rand(ar, pad(ac) + 4, device="cuda")[:, :ac]
B = torch.rand(br, pad(bc), device="cuda")[:, :bc]
C = torch.rand(m, pad(n), device="cuda")[:, :n]
os.environ.setdefault("TM_LOG", "1")
tm.sgemm_op(A, B, C, 1.5, 0.5, opa, opb, algo=algo)
torch.cuda.synchronize()
ref = 1.5 * (A.T if opa == "T" else A).double() @ (B.T if opb == "T" else B).double()
print("ok", float((C.double() - ref - 0.5 * 0).abs().max()))

import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_10694_b200 as tm
import seeded_inputs as si
A, B, C = (torch.from_numpy(x).cuda() for x in si.im2col_conv())
flush = torch.ones(512 * 2**20 // 4, device="cuda"); out = torch.empty(1, device="cuda")
def t(algo, cfg, beta=0.5):
    os.environ["TM_TC_CONFIG"] = cfg
    for _ in range(3): tm.sgemm_ex(A, B, C, 1.5, beta, algo)
    ts = []
    for _ in range(15):
        torch.sum(flush, dim=0, out=out[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); tm.sgemm_ex(A, B, C, 1.5, beta, algo); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000)
    ts.sort(); return round(ts[7], 1)
for cfg in ["2,32,0", "1,64,0", "1,32,0", "2,64,0"]:
    print(cfg, "3x", t(1, cfg), "1x", t(3, cfg), "3x beta0", t(1, cfg, 0.0))
# pure copy bandwidth reference: read A once
ts = []
for _ in range(10):
    torch.sum(flush, dim=0, out=out[0])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); s = A.sum(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1000)
ts.sort(); print("torch A.sum() us", round(ts[5], 1), "GB/s", round(A.numel() * 4 / ts[5] / 1e3, 1))

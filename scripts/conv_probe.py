"""Where does the implicit-GEMM conv spend its time?  Times variants of the
paper's Conv shape and the equivalent explicit GEMM."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_10694_b200 as tm

flush = torch.ones(512 * 2**20 // 4, device="cuda"); out = torch.empty(1, device="cuda")


def timeit(fn, reps=10):
    for _ in range(3): fn()
    ts = []
    for _ in range(reps):
        torch.sum(flush, dim=0, out=out[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort(); return ts[len(ts) // 2]


def conv(nb, h, w, c, f, r=3, beta=0.0, algo=0):
    X = torch.rand(nb, h, w, c, device="cuda"); Wt = torch.rand(f, r, r, c, device="cuda")
    Y = torch.rand(nb, h, w, f, device="cuda")
    ms = timeit(lambda: tm.conv2d_nhwc(X, Wt, Y, 1.0, beta, r // 2, algo=algo))
    byts = 4 * (X.numel() + Wt.numel() + Y.numel() * (2 if beta else 1))
    return ms, byts / ms / 1e6


mode = sys.argv[1] if len(sys.argv) > 1 else "all"
if mode == "all":
    for env in ["", "TM_KC_BLOCKS=9", "TM_KC_BLOCKS=1"]:
        subprocess.run(f"{env} python {__file__} conv", shell=True)
    subprocess.run(f"python {__file__} gemm", shell=True)
elif mode == "conv":
    tag = os.environ.get("TM_KC_BLOCKS", "-")
    for (nb, h, w, c, f) in [(32, 512, 512, 16, 16), (32, 512, 512, 32, 16), (32, 512, 512, 16, 32),
                             (32, 512, 512, 16, 64), (16, 512, 512, 64, 64)]:
        ms, gbs = conv(nb, h, w, c, f)
        print(f"kc={tag} conv N{nb} {h}x{w} C{c} F{f}: {ms:.3f} ms {gbs:.0f} GB/s", flush=True)
else:
    # explicit im2col GEMM of the same size: M = 32*512*512, N = 16, K = 144
    M, N, K = 32 * 512 * 512, 16, 144
    A = torch.rand(M, K, device="cuda"); B = torch.rand(K, N, device="cuda"); C = torch.rand(M, N, device="cuda")
    for cfg in ["1,32,0", "1,64,0", "2,32,0"]:
        os.environ["TM_TC_CONFIG"] = cfg
        ms = timeit(lambda: tm.sgemm_ex(A, B, C, 1.0, 0.0, 1))
        print(f"gemm {M}x{N}x{K} cfg {cfg}: {ms:.3f} ms {4 * (A.numel() + C.numel()) / ms / 1e6:.0f} GB/s", flush=True)
    A2 = torch.rand(M, 64, device="cuda"); B2 = torch.rand(64, 64, device="cuda"); C2 = torch.rand(M, 64, device="cuda")
    for cfg in ["1,32,0", "1,64,0", "2,32,0"]:
        os.environ["TM_TC_CONFIG"] = cfg
        ms = timeit(lambda: tm.sgemm_ex(A2, B2, C2, 1.0, 0.0, 1))
        print(f"gemm {M}x64x64 cfg {cfg}: {ms:.3f} ms {4 * (A2.numel() + C2.numel()) / ms / 1e6:.0f} GB/s", flush=True)

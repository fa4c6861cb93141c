"""How much of a small GEMM's event-timed step is the cold start after the
bench's L2 flush?  Per condition, median of 50 event-timed calls:
  flush        the bench: 512 MiB read, then start event, call, end event
  flush+touch  the same, then a one-float-per-64KiB read of A, B, C (TLB and
               page-table entries back, almost no data) before the start event
  warm         no flush (operands and translations resident); a spin kernel
               instead, so the host enqueues the call before the start event runs
for the empty elementwise launch and C2 / C4 (sgemm_ex AUTO)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1804_10694_b200 as tm

flush = torch.ones(512 * 2 ** 20 // 4, device="cuda"); fo = torch.empty(1, device="cuda")
g = torch.Generator(device="cuda"); g.manual_seed(1)


def touch(ts):
    for t in ts:
        v = t.view(-1)
        v[:: 16384].sum()


def timed(fn, ts, mode, reps=50):
    out = []
    for _ in range(reps + 5):
        if mode != "warm":
            torch.sum(flush, dim=0, out=fo[0])
        else:
            torch.cuda._sleep(200000)  # keep the GPU busy while the host enqueues (no host gap in the events)
        if mode == "flush+touch":
            touch(ts)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) * 1e3)
    out = sorted(out[5:])
    return out[len(out) // 2]


tiny = torch.zeros(1, device="cuda")
shapes = {"C2": (1060, 1060, 1060), "C4": (50176, 64, 576), "C1": (64, 64, 64)}
for mode in ("flush", "flush+touch", "warm"):
    print(f"{mode:12s} empty {timed(lambda: tiny.add_(1), [tiny], mode):7.2f} us", flush=True)
    for name, (m, n, k) in shapes.items():
        A = torch.rand(m, k, device="cuda", generator=g); B = torch.rand(k, n, device="cuda", generator=g)
        C = torch.rand(m, n, device="cuda", generator=g)
        t = timed(lambda: tm.sgemm_ex(A, B, C, 1.5, 0.5, 1), [A, B, C], mode)
        print(f"{mode:12s} {name} {t:7.2f} us", flush=True)

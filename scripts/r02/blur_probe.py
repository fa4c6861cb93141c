"""Blur bandwidth probe: tm.blur vs a plain device copy of the same bytes, at the
paper's image size and at 4x / 16x the pixels (L2 flushed before every run)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1804_10694_b200 as tm  # noqa: E402

flush = torch.ones(512 * 2 ** 20 // 4, device="cuda")
fo = torch.empty(1, device="cuda")


def timeit(fn, reps=30):
    ts = []
    for _ in range(reps + 3):
        torch.sum(flush, dim=0, out=fo[0])
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts[3:])


for (N, M) in [(2112, 3520), (4224, 7040), (8448, 14080)]:
    x = torch.rand((N, M, 3), device="cuda")
    y = torch.empty((N - 2, M - 2, 3), device="cuda")
    byts = 12 * (N * M + (N - 2) * (M - 2))
    t_blur = timeit(lambda: tm.blur(x, y))
    xs = x.view(-1)[: y.numel()]
    t_copy = timeit(lambda: y.view(-1).copy_(xs))
    print(f"{N}x{M}: blur {t_blur*1e3:.1f} us {byts/t_blur/1e6:.0f} GB/s | copy {t_copy*1e3:.1f} us "
          f"{2*y.numel()*4/t_copy/1e6:.0f} GB/s")

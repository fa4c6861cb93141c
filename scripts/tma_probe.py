"""Drive scripts/tma_probe.cu: TMA landing rate per SM for several box shapes,
issuing threads, CTAs per SM and mbarrier wait variants (random tile order)."""
import ctypes, os
import torch
here = os.path.dirname(os.path.abspath(__file__))
L = ctypes.CDLL(os.path.join(here, "libtmaprobe.so"))
big = torch.rand(2 * 2**30 // 4, device="cuda")        # 2 GiB: DRAM-resident
small = torch.rand(64 * 2**20 // 4, device="cuda")     # 64 MiB: L2-resident
WV = {0: "try_wait", 1: "test_spin", 2: "try_wait20"}
for src_name, src in [("dram", big), ("l2", small)]:
    for (mode, bc, br, swz, name) in [(0, 32, 128, 2, "2D 128Bx128 sw128"), (0, 16, 128, 1, "2D 64Bx128 sw64"),
                                      (0, 32, 32, 2, "2D 128Bx32 sw128"), (1, 2048, 1, 0, "1D bulk 8KB")]:
        cols = bc if mode == 0 else 4096
        rows = src.numel() // cols
        box_bytes = bc * br * 4
        for (stages, pairs, cps, wv) in [(8, 1, 1, 0), (8, 1, 1, 1), (8, 1, 1, 2), (8, 2, 1, 1), (16, 4, 1, 1)]:
            if stages * box_bytes * cps > 200 * 1024: continue
            loads = max(64, (src.numel() * 4 // (148 * cps)) // box_bytes) if src_name == "dram" else 1024
            loads = loads // 4 * 4
            ms = ctypes.c_float()
            rc = L.run_tma_probe(ctypes.c_void_p(src.data_ptr()), ctypes.c_longlong(rows), ctypes.c_longlong(cols),
                                 mode, bc, br, swz, stages, loads, pairs, cps, wv, ctypes.byref(ms))
            byts = 148 * cps * loads * box_bytes
            print(f"{src_name:4s} {name:18s} st{stages:2d} issuers{pairs} ctas/SM{cps} {WV[wv]:10s} rc{rc} "
                  f"{ms.value*1e3:8.1f} us {byts/ms.value/1e6:7.0f} GB/s {ms.value*1e6/(loads*cps):6.1f} ns/load/SM",
                  flush=True)

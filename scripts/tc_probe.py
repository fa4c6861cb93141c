import ctypes
import os
import sys

import numpy as np
import torch

np.set_printoptions(linewidth=220, precision=2, suppress=True)
here = os.path.dirname(os.path.abspath(__file__))
L = ctypes.CDLL(os.path.join(here, "libtcprobe.so"))
vp = ctypes.c_void_p


class Cfg(ctypes.Structure):
    _fields_ = [("a_mode", ctypes.c_int), ("b_mode", ctypes.c_int)] + [
        (n, ctypes.c_uint32) for n in ("a_lbo", "a_sbo", "a_layout", "b_lbo", "b_sbo", "b_layout", "idesc")]


def idesc(amn, bmn, M=128, N=32):
    return (1 << 4) | (2 << 7) | (2 << 10) | (amn << 15) | (bmn << 16) | ((N >> 3) << 17) | ((M >> 4) << 24)


g = np.random.default_rng(0)
A = g.integers(-3, 4, (128, 8)).astype(np.float32)
B = g.integers(-3, 4, (8, 32)).astype(np.float32)
E = A @ B
dA = torch.from_numpy(A).cuda()
dB = torch.from_numpy(B).cuda()
cases = []
# (name, a_mode, b_mode, a_lbo, a_sbo, a_layout, b_lbo, b_sbo, b_layout, amn, bmn)
cases.append(("ref none/none", 0, 0, 128, 256, 0, 128, 256, 0, 0, 0))
for a_lbo in (16, 0, 128):
    cases.append((f"A sw128 lbo{a_lbo} / B none", 1, 0, a_lbo, 1024, 2, 128, 256, 0, 0, 0))
for (bl, bs) in [(4096, 1024), (1024, 4096), (0, 1024), (1024, 0), (16, 1024), (1024, 16)]:
    cases.append((f"A none / B MN sw128 lbo{bl} sbo{bs}", 0, 1, 128, 256, 0, bl, bs, 2, 0, 1))
for (bl, bs) in [(4096, 512), (512, 4096), (16, 512), (4096, 1024), (4096, 128)]:
    cases.append((f"A none / B MN sw128_32B lbo{bl} sbo{bs}", 0, 3, 128, 256, 0, bl, bs, 1, 0, 1))
for (bl, bs) in [(1024, 128), (128, 1024), (128, 128)]:
    cases.append((f"A none / B MN none lbo{bl} sbo{bs}", 0, 2, 128, 256, 0, bl, bs, 0, 0, 1))
for c in cases:
    name, am, bm, al, asb, alay, bl, bs, blay, amn, bmn = c
    cfg = Cfg(am, bm, al, asb, alay, bl, bs, blay, idesc(amn, bmn))
    dO = torch.full((128, 32), -7.0, device="cuda")
    rc = L.run_probe_mma(vp(dA.data_ptr()), vp(dB.data_ptr()), vp(dO.data_ptr()), ctypes.byref(cfg))
    O = dO.cpu().numpy()
    ok = np.isclose(O, E).mean()
    print(f"{name:45s} rc {rc} ok {ok*100:.1f}%  O[0,:6]={O[0,:6]}")
print("E[0,:6]", E[0, :6])

# ---- bf16 kind::f16: does MN-major B work there?
def idesc16(amn, bmn, M=128, N=32):
    return (1 << 4) | (1 << 7) | (1 << 10) | (amn << 15) | (bmn << 16) | ((N >> 3) << 17) | ((M >> 4) << 24)

A16 = g.integers(-3, 4, (128, 16)).astype(np.float32)
B16 = g.integers(-3, 4, (16, 32)).astype(np.float32)
E16 = A16 @ B16
tA = torch.from_numpy(A16).to(torch.bfloat16).cuda().view(torch.int16)
tB = torch.from_numpy(B16).to(torch.bfloat16).cuda().view(torch.int16)
for name, bm, bl, bs, blay, bmn in [("bf16 B K-major none", 0, 128, 256, 0, 0),
                                    ("bf16 B MN none lbo512 sbo128", 2, 512, 128, 0, 1),
                                    ("bf16 B MN none lbo128 sbo512", 2, 128, 512, 0, 1),
                                    ("bf16 B MN sw128 lbo4096 sbo1024", 1, 4096, 1024, 2, 1),
                                    ("bf16 B MN sw128 lbo1024 sbo4096", 1, 1024, 4096, 2, 1)]:
    cfg = Cfg(0, bm, 128, 256, 0, bl, bs, blay, idesc16(0, bmn))
    dO = torch.full((128, 32), -7.0, device="cuda")
    rc = L.run_probe_mma_bf16(vp(tA.data_ptr()), vp(tB.data_ptr()), vp(dO.data_ptr()), ctypes.byref(cfg))
    O = dO.cpu().numpy()
    print(f"{name:45s} rc {rc} ok {np.isclose(O, E16).mean()*100:.1f}%  O[0,:6]={O[0,:6]} E={E16[0,:6]}")

# ---- tf32 A MN-major (transpose A) with B K-major

"""Drive tmem_contention.cu: tcgen05.mma kind::tf32 cycles per MMA (A in TMEM)
alone, beside a warpgroup storing to TMEM (tcgen05.st.32x32b.x32 + wait), and
beside one loading from TMEM (tcgen05.ld.32x32b.x16 + wait)."""
import ctypes, os
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtmemcont.so"))
for n in (48, 96, 144):
    for mode, name in ((0, "alone"), (1, "beside tcgen05.st"), (2, "beside tcgen05.ld"), (3, "beside ld.shared"), (4, "st into A columns"), (5, "conv tile chain"), (6, "conv chain+commit"), (7, "+FFMA same SMSP"), (8, "+FFMA other SMSP"), (9, "lean loop+FFMA same")):
        c, o = ctypes.c_ulonglong(), ctypes.c_ulonglong()
        rc = L.run_cont(n, 8160 if mode >= 5 else 8192, mode, ctypes.byref(c), ctypes.byref(o))
        print(f"N={n:3d} {name:18s} rc={rc}: {c.value / (8160 if mode >= 5 else 8192):6.1f} cycles per MMA (side ops {o.value})", flush=True)

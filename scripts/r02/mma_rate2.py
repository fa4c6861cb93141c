"""tcgen05 kind::tf32 cycles per MMA for the direct-conv configuration (A from
TMEM, B SWIZZLE_64B) next to the GEMM's (A from smem, B SW128); drives
scripts/mma_rate.cu (build: see its header)."""
import ctypes, os
here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = ctypes.CDLL(os.path.join(here, "libmmarate.so"))


def run(n, a_tmem=0, reps=4096, n_acc=0, m=128, bsw=128):
    ic, tc, ms = ctypes.c_ulonglong(), ctypes.c_ulonglong(), ctypes.c_float()
    rc = L.run_mma_rate(n, a_tmem, reps, n_acc, m, bsw, ctypes.byref(ic), ctypes.byref(tc), ctypes.byref(ms))
    cyc = tc.value / reps
    print(f"M={m} N={n:3d} A={'tmem' if a_tmem else 'smem'} Bsw={bsw} accs={n_acc} rc={rc}: issue "
          f"{ic.value/reps:6.1f}, total {cyc:6.1f} cyc/MMA -> {m*n*8/cyc:7.1f} MAC/clk/SM", flush=True)


for bsw in (128, 64):
    for a in (0, 1):
        for n in (32, 48, 64, 80, 96, 112, 128, 144, 192, 256):
            run(n, a_tmem=a, bsw=bsw)
for n in (48, 96):
    run(n, a_tmem=1, bsw=64, n_acc=-2)
    run(n, a_tmem=1, bsw=64, n_acc=-1)

"""Drive scripts/mma_rate.cu: tcgen05 kind::tf32 (cta_group::1) cycles per MMA vs M, N, A source, burst length."""
import ctypes, os
here = os.path.dirname(os.path.abspath(__file__))
L = ctypes.CDLL(os.path.join(here, "libmmarate.so"))


def run(n, a_tmem=0, reps=4096, n_acc=1, m=128, bsw=128):
    ic, tc, ms = ctypes.c_ulonglong(), ctypes.c_ulonglong(), ctypes.c_float()
    rc = L.run_mma_rate(n, a_tmem, reps, n_acc, m, bsw, ctypes.byref(ic), ctypes.byref(tc), ctypes.byref(ms))
    cyc = tc.value / reps
    print(f"M={m} N={n:3d} A={'tmem' if a_tmem else 'smem'} Bsw={bsw} accs={n_acc} reps={reps} rc={rc}: issue "
          f"{ic.value/reps:6.1f}, total {cyc:6.1f} cyc/MMA, kernel {ms.value*1e3:8.1f} us -> "
          f"{m*n*8/cyc:7.1f} MAC/clk/SM", flush=True)


print("-- lean issue loop (loop-invariant operands, 8 MMAs per iteration): tensor throughput")
for a in (0, 1):
    for n in (16, 32, 48, 64, 96, 128, 192, 256):
        run(n, a_tmem=a, n_acc=0)
print("-- same arithmetic, whole warp in the loop, elected lane issues")
for n in (48, 256):
    run(n, n_acc=-1)
    run(n, n_acc=-1, a_tmem=1)
print("-- per-MMA address arithmetic in the loop (modulo, R2UR): issue-bound")
for n in (48, 256):
    run(n, n_acc=1)

import ctypes, os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_10694_b200 as tm
s = 64
A = torch.rand(s, s, device="cuda"); B = torch.rand(s, s, device="cuda"); C = torch.rand(s, s, device="cuda")
def bench(fn, n=2000):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    t1 = time.perf_counter(); torch.cuda.synchronize()
    return (t1 - t0) / n * 1e6
vp = ctypes.c_void_p
args = (s, s, s, 1.5, vp(A.data_ptr()), s, vp(B.data_ptr()), s, 0.5, vp(C.data_ptr()), s, vp(0))
print("python sgemm_ex tc  us/call", round(bench(lambda: tm.sgemm_ex(A, B, C, 1.5, 0.5, 1)), 2))
print("python sgemm_ex simt us/call", round(bench(lambda: tm.sgemm_ex(A, B, C, 1.5, 0.5, 2)), 2))
print("ctypes raw tc       us/call", round(bench(lambda: tm.lib.tm_sgemm_ex(*args, 1)), 2))
print("ctypes raw simt     us/call", round(bench(lambda: tm.lib.tm_sgemm_ex(*args, 2)), 2))
print("ctypes plan_name    us/call", round(bench(lambda: tm.lib.tm_sgemm_plan_name(*args[:-1], 1)), 2))
print("torch current_stream us/call", round(bench(lambda: torch.cuda.current_stream().cuda_stream), 2))
print("torch mm 64 us/call", round(bench(lambda: torch.mm(A, B, out=C)), 2))

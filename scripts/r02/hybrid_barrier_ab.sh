# Hybrid stream-K + wave barrier over the data-parallel waves: C3 with the barrier on/off,
# and one P = 8 rank of C5 (2048 x 16384 x 16384) hybrid (2,128,1) vs data-parallel (2,128,0).
timeout 600 python -m pytest tests/test_graphs.py tests/test_parity.py -q -x -p no:cacheprovider -k "graph or streamk or c3" 2>&1 | tail -2
for i in 1 2; do
  for w in 1 0; do TM_WAVE_SYNC=$w bash scripts/ms.sh "C3 wave_sync=$w" --config C3 --steps 30 --warmup 5 --no-cpu --no-e2e; done
done
python - <<'PY'
import os, statistics, sys, time
import torch
sys.path.insert(0, ".")
import paper_1804_10694_b200 as tm
S = 16384
g = torch.Generator(device="cuda").manual_seed(5)
A = torch.rand(2048, S, device="cuda", generator=g); B = torch.rand(S, S, device="cuda", generator=g)
C = torch.rand(2048, S, device="cuda", generator=g)
def soak(fn, seconds=1.5, reps=7):
    t0 = time.time()
    while time.time() - t0 < seconds:
        fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return round(statistics.median(ts), 3)
for rep in range(2):
    for cfg in ("2,128,0", "2,128,1"):
        os.environ["TM_TC_CONFIG"] = cfg
        print(f"P=8 rank 2048x16384x16384 cfg {cfg}: {soak(lambda: tm.sgemm_ex(A, B, C, 1.5, 0.5))} ms", flush=True)
PY

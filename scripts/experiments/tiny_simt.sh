for c in C1; do
bash scripts/ms.sh "$c tc" --config $c --steps 30 --warmup 5 --no-cpu --no-e2e
bash scripts/ms.sh "$c simt" --config $c --algo simt --steps 30 --warmup 5 --no-cpu --no-e2e
done
python - <<'PY'
import torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_1804_10694_b200 as tm
flush = torch.ones(512 * 2**20 // 4, device="cuda"); out = torch.empty(1, device="cuda")
for s in (32, 64, 128, 192, 256, 384, 512):
    A = torch.rand(s, s, device="cuda"); B = torch.rand(s, s, device="cuda"); C = torch.rand(s, s, device="cuda")
    res = []
    for algo in (1, 2):
        ts = []
        for i in range(25):
            torch.sum(flush, dim=0, out=out[0])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); tm.sgemm_ex(A, B, C, 1.5, 0.5, algo); e1.record(); torch.cuda.synchronize()
            if i >= 5: ts.append(e0.elapsed_time(e1) * 1000)
        ts.sort(); res.append(round(ts[len(ts)//2], 1))
    print(s, "tc", res[0], "simt", res[1], "auto plan", tm.plan_config(s, s, s, 1.5, 0.5))
PY

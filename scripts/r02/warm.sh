# L2 warm-up of small problems on/off (TM_L2_WARM), event-timed bench lines and a C2 timeline.
set -u
timeout 900 python -m pytest tests/test_parity.py tests/test_transposes.py -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -2
for w in 1 0 1 0; do
  for c in C2 C3; do TM_L2_WARM=$w timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c warm=$w', d['step_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
done
for sz in 512 768 2048; do for w in 1 0; do TM_L2_WARM=$w python - <<PY
import os, sys, statistics, torch
sys.path.insert(0, ".")
import paper_1804_10694_b200 as tm
flush = torch.ones(512 * 2 ** 20 // 4, device="cuda"); fo = torch.empty(1, device="cuda")
S = $sz
A, B, C = (torch.rand(S, S, device="cuda") for _ in range(3))
ts = []
for i in range(40):
    torch.sum(flush, dim=0, out=fo[0])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); tm.sgemm_ex(A, B, C, 1.5, 0.5, 1); e1.record(); torch.cuda.synchronize()
    if i >= 5: ts.append(e0.elapsed_time(e1) * 1000)
print("S", S, "warm", os.environ["TM_L2_WARM"], round(statistics.median(ts), 2), "us")
PY
done; done
rm -f /tmp/trw.jsonl
TM_L2_WARM=1 python scripts/r02/trace_c2.py /tmp/trw.jsonl 2,64,1/0.5
python scripts/trace_report.py /tmp/trw.jsonl | grep -E "setup_done|first_stage|first_mma |last_mma|epilogue_done|teardown"

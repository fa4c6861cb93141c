# C2 / C4 / C3: cooperative launch attribute on vs off (same kernel), first-stage latency.
set -u
for c in C2 C4 C3; do
  for coop in 1 0; do
    TM_COOPERATIVE=$coop timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c coop=$coop', d['step_ms'], d['roofline']['frac'])"
  done
done
rm -f /tmp/trc.jsonl
TM_COOPERATIVE=0 python scripts/r02/trace_c2.py /tmp/trc.jsonl 2,64,1/0.5
python scripts/trace_report.py /tmp/trc.jsonl | grep -E "setup_done|first_stage|first_mma|epilogue_done|teardown"

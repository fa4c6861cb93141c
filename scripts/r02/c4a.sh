# C4 (conv-shaped 50176x64x576): configs, a per-CTA timeline; conv 7x7 direct.
set -u
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_conv.py -q -p no:cacheprovider --timeout 300 -k "direct or 9x9" 2>&1 | tail -2
for r in 5 7; do timeout 300 python bench.py --config CONV --conv-r $r --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('conv r', $r, d['ms_per_step'], d['value'], d['roofline']['kernel'])"; done
for cfg in auto 2,32,1 2,32,0 2,64,1 1,64,1 1,32,1 1,128,1; do
  if [ $cfg = auto ]; then unset TM_TC_CONFIG; else export TM_TC_CONFIG=$cfg; fi
  timeout 300 python bench.py --config C4 --steps 50 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4', '$cfg', d['step_ms'], d['roofline']['frac'])"
done
unset TM_TC_CONFIG
rm -f /tmp/tr4.jsonl
TM_TRACE_PATH=/tmp/tr4.jsonl python bench.py --config C4 --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1
python scripts/trace_report.py /tmp/tr4.jsonl | tail -40

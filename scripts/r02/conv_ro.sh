# Two output rows per tile (default for N_row <= 48) vs one (TM_CONV_RO=1): parity, bench, role stats.
set -u
timeout 900 python -m pytest tests/test_conv.py -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -3
TM_CONV_RO=1 timeout 900 python -m pytest tests/test_conv.py -q -p no:cacheprovider --timeout 600 -x -k "direct or paper" 2>&1 | tail -2
for rep in 1 2; do
for ro in 2 1; do
  for cfg in "--conv-r 3" "--conv-r 3 --conv-beta 0.5" "--conv-valid"; do
    TM_CONV_RO=$ro timeout 300 python bench.py --config CONV $cfg --steps 20 --warmup 5 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('ro=$ro $cfg', d['ms_per_step'], r['frac'], d['clocks']['sm_mhz'])"
  done
done
done
rm -f /tmp/cs.jsonl
TM_CONV_STATS=/tmp/cs.jsonl python bench.py --config CONV --conv-r 3 --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1; head -1 /tmp/cs.jsonl

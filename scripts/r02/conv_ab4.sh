set -u
for rep in 1 2; do
for pad in 0 20480; do
  for r in 9 11; do TM_CONV_SMEMPAD=$pad timeout 300 python bench.py --config CONV --conv-r $r --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('pad=$pad conv r', $r, d['ms_per_step'], r['frac'], d['clocks']['sm_mhz'])"; done
done
(cd _ab_old && for r in 9; do timeout 300 python bench.py --config CONV --conv-r $r --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('old conv r', $r, d['ms_per_step'], r['frac'], d['clocks']['sm_mhz'])"; done)
done

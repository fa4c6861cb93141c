set -u
timeout 900 python -m pytest tests/test_conv.py -q -p no:cacheprovider --timeout 600 2>&1 | tail -3
for nm in 0 1; do
  if [ $nm = 1 ]; then export TM_CONV_NOMERGE=1; else unset TM_CONV_NOMERGE; fi
  for r in 1 3 5 7; do timeout 300 python bench.py --config CONV --conv-r $r --steps 20 --warmup 5 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('nomerge=$nm conv r', $r, d['ms_per_step'], r['bound'], r['frac'], r.get('hbm_frac'), d['clocks']['sm_mhz'])"; done
done

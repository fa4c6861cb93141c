# A/B on one box: before the two-row tiles (_ab_old = 6e9d677) vs HEAD, 9x9 / 11x11 / 7x7.
set -u
for rep in 1 2; do
for tree in _ab_old .; do
  (cd $tree && for r in 9 11 7; do timeout 300 python bench.py --config CONV --conv-r $r --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$tree conv r', $r, d['ms_per_step'], r['frac'], d['clocks']['sm_mhz'])"; done)
done
done

# A/B: the committed conv kernel (_ab_old, git worktree of HEAD) vs the working tree, same box.
set -u
for rep in 1 2; do
for tree in _ab_old .; do
  (cd $tree && for r in 3 5; do timeout 300 python bench.py --config CONV --conv-r $r --steps 20 --warmup 5 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$tree conv r', $r, d['ms_per_step'], r['frac'], d['clocks']['sm_mhz'])"; done)
done
done

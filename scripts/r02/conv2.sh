set -u
timeout 900 python -m pytest tests/test_conv.py -q -p no:cacheprovider --timeout 600 2>&1 | tail -4
for r in 3 5 7 9 11; do timeout 300 python bench.py --config CONV --conv-r $r --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('conv r', $r, d['ms_per_step'], d['gflops'], r['bound'], r['frac'], r['kernel'])"; done

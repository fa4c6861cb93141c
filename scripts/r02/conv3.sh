set -u
timeout 900 python -m pytest tests/test_conv.py tests/test_blur.py -q -p no:cacheprovider --timeout 600 2>&1 | tail -3
for r in 3 5 9; do timeout 300 python bench.py --config CONV --conv-r $r --steps 20 --warmup 5 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('conv r', $r, d['ms_per_step'], r['bound'], r['frac'], r.get('hbm_frac'), d['clocks']['sm_mhz'])"; done
timeout 300 python bench.py --config CONV --conv-beta 0.5 --steps 20 --warmup 5 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('conv beta', d['ms_per_step'], r['frac'], d['clocks']['sm_mhz'])"
timeout 300 python bench.py --config BLUR --steps 20 --warmup 5 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('blur', d['step_ms'], d['roofline']['frac'])"

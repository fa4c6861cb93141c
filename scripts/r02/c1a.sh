set -u
timeout 600 python -m pytest tests/test_small.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -2
for i in 1 2 3; do timeout 300 python bench.py --config C1 --steps 100 --warmup 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1', d['step_ms'])"; done

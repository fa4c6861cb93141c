timeout 600 python -m pytest tests/test_parity.py -q -m gpu -p no:cacheprovider -x -k host 2>&1 | tail -2
python bench.py --config C5 --steps 3 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C5 value', d['value'], 'e2e', d['e2e'])"
python bench.py --config C3b --steps 3 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C3b value', d['value'], 'e2e', d['e2e'])"

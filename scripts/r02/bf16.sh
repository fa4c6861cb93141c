set -u
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_bf16x9.py -q -p no:cacheprovider --timeout 300 -x 2>&1 | tail -15
timeout 300 python bench.py --config C3b --algo bf16x9 --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-1200

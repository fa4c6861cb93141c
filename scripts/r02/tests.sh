set -u
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests/ -m gpu -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -15
for c in C2 C4; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-1500; done

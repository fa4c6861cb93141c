set -u
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests/ -m gpu -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -4
python scripts/r02/small_probe.py 2>&1 | tee gpurun_out/small_probe_r02b.txt
for c in C1 C2; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-400; done

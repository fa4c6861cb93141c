set -u
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_small.py tests/test_parity.py -m gpu -q -p no:cacheprovider --timeout 300 -x -k "small or auto or c1" 2>&1 | tail -5
python scripts/r02/small_probe.py 2>&1 | tee gpurun_out/small_probe_r02.txt
timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-700

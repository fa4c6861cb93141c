# Re-entry check at HEAD: smoke, every GPU test, the default bench line.
set -u
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 1500 python -m pytest tests/ -m gpu -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/bench_verify.json 2> gpurun_out/bench_verify.err; tail -1 gpurun_out/bench_verify.json | cut -c1-400
for c in C1 C2 C4; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | cut -c1-200; done
timeout 300 python bench.py --config CONV --steps 20 --warmup 5 --no-cpu 2>/dev/null | tail -1 | cut -c1-200

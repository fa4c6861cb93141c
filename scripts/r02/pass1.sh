# Round-2 session-2 first GPU pass at HEAD: smoke, all GPU tests, default bench, config lines.
set -u
TAG=r02b
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests/ -m gpu -q -p no:cacheprovider --timeout 600 2>&1 | tail -25 > gpurun_out/gputests_$TAG.txt
cat gpurun_out/gputests_$TAG.txt | tail -8
timeout 600 python bench.py 2>gpurun_out/bench_default_$TAG.err | tail -1 > gpurun_out/bench_default_$TAG.json
cut -c1-600 gpurun_out/bench_default_$TAG.json
for c in C1 C2 C3 C4 CONV; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1; done > gpurun_out/bench_configs_$TAG.jsonl
cut -c1-300 gpurun_out/bench_configs_$TAG.jsonl

# bench_configs lines only (the configs part of scripts/gpu_full.sh)
TAG=${TAG:-r01}
for c in C1 C2 C3 C3b C4; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1; done > gpurun_out/bench_configs_$TAG.jsonl
timeout 300 python bench.py --config C3 --algo simt --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 >> gpurun_out/bench_configs_$TAG.jsonl
timeout 300 python bench.py --config C3b --algo tf32x1 --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 >> gpurun_out/bench_configs_$TAG.jsonl
timeout 300 python bench.py --config CONV --steps 20 --warmup 5 --no-cpu 2>/dev/null | tail -1 >> gpurun_out/bench_configs_$TAG.jsonl
timeout 300 python bench.py --config CONV --conv-beta 0.5 --steps 20 --warmup 5 --no-cpu 2>/dev/null | tail -1 >> gpurun_out/bench_configs_$TAG.jsonl

# Full GPU pass: smoke, tests, default bench line, per-config lines, ncu evidence.
set -u
TAG=${TAG:-r01}
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests/ -m gpu -q -p no:cacheprovider --timeout 300 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err; tail -1 gpurun_out/bench_default_$TAG.json
for c in C1 C2 C3 C3b C4; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1; done > gpurun_out/bench_configs_$TAG.jsonl
timeout 300 python bench.py --config C3 --algo simt --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 >> gpurun_out/bench_configs_$TAG.jsonl
timeout 300 python bench.py --config C3b --algo tf32x1 --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 >> gpurun_out/bench_configs_$TAG.jsonl
timeout 300 python bench.py --config CONV --steps 20 --warmup 5 --no-cpu 2>/dev/null | tail -1 >> gpurun_out/bench_configs_$TAG.jsonl
timeout 300 python bench.py --config CONV --conv-beta 0.5 --steps 20 --warmup 5 --no-cpu 2>/dev/null | tail -1 >> gpurun_out/bench_configs_$TAG.jsonl
cut -c1-200 gpurun_out/bench_configs_$TAG.jsonl
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_$TAG.json 2>&1; tail -1 gpurun_out/bench_reference_$TAG.json | cut -c1-300
TM_COOPERATIVE=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
TM_COOPERATIVE=0 ncu --set full --clock-control none --import-source on -k regex:k_sgemm_tc -s 3 -c 1 -o gpurun_out/prof_c5_$TAG python bench.py --config C5 --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
TM_COOPERATIVE=0 ncu --set full --clock-control none --import-source on -k regex:k_sgemm_tc -s 3 -c 1 -o gpurun_out/prof_c4_$TAG python bench.py --config C4 --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
TM_COOPERATIVE=0 ncu --set full --clock-control none --import-source on -k regex:k_sgemm_simt -s 2 -c 1 -o gpurun_out/prof_simt_c3_$TAG python bench.py --config C3 --algo simt --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_conv_direct -s 1 -c 1 -o gpurun_out/prof_conv_$TAG python bench.py --config CONV --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ls gpurun_out | grep $TAG

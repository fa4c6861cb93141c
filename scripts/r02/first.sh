# Round-2 first GPU pass: tests green at HEAD, config lines, ncu full on C2 and C1.
set -u
TAG=r02a
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests/ -m gpu -q -p no:cacheprovider --timeout 300 2>&1 | tail -3
for c in C1 C2 C4; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1; done > gpurun_out/bench_configs_$TAG.jsonl
cut -c1-400 gpurun_out/bench_configs_$TAG.jsonl
for c in C1 C2; do
  ncu --set full --clock-control none --import-source on -k regex:k_sgemm -s 3 -c 1 -o gpurun_out/prof_${c}_$TAG python bench.py --config $c --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${c}_$TAG.csv python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
ls gpurun_out | grep $TAG

timeout 900 python -m pytest tests/ -m gpu -q -p no:cacheprovider --timeout 600 2>&1 | tail -8
for c in C5 C3b C3 C4 C2; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], 'ms', d['value'], 'GF/s', d['roofline']['frac'], d['config']['path'], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; done
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench_default.json; cat gpurun_out/bench_default.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sgemm_tc -s 3 -c 1 -o gpurun_out/prof_c5_r01c python bench.py --config C5 --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ls gpurun_out

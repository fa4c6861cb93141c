# quick perf + correctness check
timeout 600 python -m pytest tests/ -m gpu -q -p no:cacheprovider --timeout 300 -x 2>&1 | tail -3
for c in ${CONFIGS:-C5 C3b C3 C4 C2}; do timeout 300 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], 'ms', d['value'], 'GF/s', d['roofline']['frac'], d['config']['path'], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; done

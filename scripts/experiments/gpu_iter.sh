# one GPU iteration: parity tests, accuracy survey, benches
timeout 600 python -m pytest tests/test_parity.py tests/test_probes.py -q -p no:cacheprovider --timeout 300 -x 2>&1 | tail -15
timeout 600 python scripts/accuracy.py 2>&1 | tail -4
for c in C5 C3b C3 C4 C2; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], 'ms', d['value'], 'GF/s', d['roofline']['frac'], d['config']['path'], d['clocks'].get('sm_mhz'))"; done

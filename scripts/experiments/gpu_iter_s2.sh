# iteration check: GPU parity tests (-x) + per-config times and a C2/C4 trace
timeout 900 python -m pytest tests/ -m gpu -q -p no:cacheprovider --timeout 300 -x 2>&1 | tail -2
for c in ${CONFIGS:-C1 C2 C4 C3 C3b}; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], 'ms', d['value'], 'GF/s', d['roofline']['frac'], d['config']['path'])"; done
rm -f /tmp/tr.jsonl
for c in C2 C4; do TM_TRACE_PATH=/tmp/tr.jsonl python bench.py --config $c --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1; done
cp /tmp/tr.jsonl gpurun_out/trace_iter.jsonl

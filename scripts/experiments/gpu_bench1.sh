set -x
nproc
timeout 600 python scripts/accuracy.py 2>&1 | tail -8
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | tail -5
for c in C3 C3b C4 C2; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -2; done
timeout 300 python bench.py --config C3 --algo simt --steps 5 --warmup 2 --no-cpu --no-e2e 2>&1 | tail -2
for cfg in 2,128 2,64 1,128 1,64; do TM_TC_CONFIG=$cfg timeout 300 python bench.py --config C3b --steps 5 --warmup 2 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['roofline']['frac'])"; done

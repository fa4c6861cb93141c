for c in C1 C2 C4; do python bench.py --config $c --steps 5 --warmup 3 --no-e2e 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c', d['cpu_baseline'])"; done
python bench.py --config C3b --algo tf32x1 --steps 3 --warmup 3 --no-e2e 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C3b x1', d['cpu_baseline'])"
time python bench.py --steps 3 --warmup 3 --no-e2e 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C5', d['cpu_baseline'])"

rm -f /tmp/tr.jsonl
for cfg in 2,128,1 2,64,1 2,64,0; do TM_TC_CONFIG=$cfg TM_TRACE_PATH=/tmp/tr.jsonl python bench.py --config C2 --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1; done
cp /tmp/tr.jsonl gpurun_out/trace4.jsonl
python scripts/trace_report.py /tmp/tr.jsonl
for i in 1 2 3; do for cfg in 2,128,1 2,64,0 1,128,0; do TM_TC_CONFIG=$cfg python bench.py --config C2 --steps 20 --warmup 5 --no-cpu --no-e2e | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(\"C2 $cfg\", d[\"ms_per_step\"], d[\"roofline\"][\"frac\"])"; done; done

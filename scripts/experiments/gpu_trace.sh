rm -f /tmp/tr.jsonl
for cfg in 2,128,0 2,64,0 1,128,0; do TM_TC_CONFIG=$cfg TM_TRACE_PATH=/tmp/tr.jsonl python bench.py --config C2 --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1; done
TM_TRACE_PATH=/tmp/tr.jsonl python bench.py --config C4 --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1
TM_TRACE_PATH=/tmp/tr.jsonl python bench.py --config C3 --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1
cp /tmp/tr.jsonl gpurun_out/trace1.jsonl
python scripts/trace_report.py /tmp/tr.jsonl

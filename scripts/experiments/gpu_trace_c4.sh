rm -f /tmp/tr.jsonl
for cfg in 2,32,0 2,32,1; do TM_TC_CONFIG=$cfg TM_TRACE_PATH=/tmp/tr.jsonl python bench.py --config C4 --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1; done
cp /tmp/tr.jsonl gpurun_out/trace_c4.jsonl

rm -f /tmp/tr.jsonl
TM_TRACE_PATH=/tmp/tr.jsonl python bench.py --config C1 --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1
TM_TRACE_PATH=/tmp/tr.jsonl python bench.py --config C2 --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1
for cfg in 1,64,0 2,64,0 1,64,1; do TM_TC_CONFIG=$cfg TM_TRACE_PATH=/tmp/tr.jsonl python bench.py --config C2 --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1; done
TM_TC_CONFIG=2,32,0 TM_TRACE_PATH=/tmp/tr.jsonl python bench.py --config C4 --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1
cp /tmp/tr.jsonl gpurun_out/trace_s2b.jsonl
for cfg in 2,64,1 1,64,0 2,64,0 1,64,1 1,128,1 2,128,1 1,32,1; do echo $cfg; TM_TC_CONFIG=$cfg python bench.py --config C2 --steps 20 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | cut -c1-200; done

# C4 / C2 timelines (TM_TRACE_PATH) and the C4 config probe
rm -f /tmp/tr.jsonl
for c in C4 C2; do TM_TRACE_PATH=/tmp/tr.jsonl python bench.py --config $c --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1; done
TM_TC_CONFIG=1,64,0 TM_TRACE_PATH=/tmp/tr.jsonl python bench.py --config C4 --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1
TM_TC_CONFIG=2,32,0 TM_TRACE_PATH=/tmp/tr.jsonl python bench.py --config C4 --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1
cp /tmp/tr.jsonl gpurun_out/trace_s2.jsonl
python scripts/c4_probe.py

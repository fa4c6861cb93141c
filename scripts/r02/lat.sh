set -u
python scripts/r02/latency_probe.py 2>&1 | tee gpurun_out/latency_probe_r02.txt
rm -f /tmp/tr.jsonl
TM_TRACE_PATH=/tmp/tr.jsonl python bench.py --config C1 --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1
for cfg in 2,64,1 2,128,1 1,128,1; do TM_TC_CONFIG=$cfg TM_TRACE_PATH=/tmp/tr.jsonl python bench.py --config C2 --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1; done
python scripts/trace_report.py /tmp/tr.jsonl | tee gpurun_out/trace_small_r02.txt
TM_COOPERATIVE=0 ncu --set full --clock-control none --import-source on -k regex:k_sgemm -s 3 -c 1 -o gpurun_out/prof_C2_r02a python bench.py --config C2 --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
TM_COOPERATIVE=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2_r02a.csv python bench.py --config C2 --steps 5 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1

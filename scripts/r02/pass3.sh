set -u
timeout 1500 python -m pytest tests/test_parity.py tests/test_transposes.py tests/test_blur.py tests/test_graphs.py tests/test_tf32x1.py tests/test_bf16x9.py -q -p no:cacheprovider --timeout 600 2>&1 | tail -3
for c in C5 C3b C3; do timeout 300 python bench.py --config $c --steps 10 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['step_ms']['median'], d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
TM_COOPERATIVE=0 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_sgemm_tc -s 3 -c 1 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "dram__|duration"

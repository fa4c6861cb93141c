# Blur v2 (shuffle + prefetch ring): parity, strip-height sweep, launch list.
set -u
timeout 600 python -m pytest tests/test_blur.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -4
for rb in 16 32 64 128 256; do echo "rb=$rb"; TM_BLUR_RB=$rb timeout 300 python bench.py --config BLUR --steps 50 --warmup 5 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['step_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
timeout 300 python bench.py --config BLUR --steps 50 --warmup 5 2>&1 | tail -1 > gpurun_out/bench_blur_r02.json
cut -c1-400 gpurun_out/bench_blur_r02.json
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_blur_r02.csv python bench.py --config BLUR --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1
grep k_blur gpurun_out/launches_blur_r02.csv | head -3 | cut -c 1-40,180-

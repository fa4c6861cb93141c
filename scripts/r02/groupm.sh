# Grouped-raster height (TM_GROUP_M, tiles) vs sustained C5 / C3b throughput.
set -u
for gm in 16 8 10 12 6; do
  for c in C5 C3b; do
    TM_GROUP_M=$gm timeout 300 python bench.py --config $c --steps 10 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gm', $gm, '$c', d['step_ms']['median'], d['value'], d['roofline']['frac'], d['roofline'].get('frac_clock_normalized'), d['clocks']['sm_mhz'])"
  done
done
TM_GROUP_M=8 TM_COOPERATIVE=0 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_sgemm_tc -s 3 -c 1 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "dram__|duration" 

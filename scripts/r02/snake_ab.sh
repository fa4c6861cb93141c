# A/B: snake K order across data-parallel waves (TM_SNAKE_K=1) vs forward (0): C5 / C3b
# throughput (interleaved, soaked) and C5 DRAM bytes per launch (ncu, one launch each).
timeout 300 python -m pytest tests/test_parity.py -q -x -p no:cacheprovider -k "c3b or large_k or deterministic" 2>&1 | tail -1
TM_SNAKE_K=1 timeout 300 python -m pytest tests/test_parity.py -q -x -p no:cacheprovider -k "c3b or large_k or deterministic" 2>&1 | tail -1
for i in 1 2; do
  for sn in 0 1; do
    TM_SNAKE_K=$sn bash scripts/ms.sh "C5 snake=$sn" --steps 10 --warmup 3 --no-cpu --no-e2e
    TM_SNAKE_K=$sn bash scripts/ms.sh "C3b snake=$sn" --config C3b --steps 20 --warmup 3 --no-cpu --no-e2e
  done
done
for sn in 0 1; do
  TM_SNAKE_K=$sn TM_COOPERATIVE=0 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_sgemm_tc -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "dram__|gpu__time" | sed "s/^/snake=$sn /"
done

# GEMM: barriers right after the epilogue staging (product) vs 8 KiB further (-DTM_BAR_PAD=8192 build in _exp/).
set -u
for rep in 1 2; do
for lib in "" _exp/libtm_pad8k.so; do
  for c in C2 C4 C3 C3b; do
    TM_LIB_PATH=${lib:-paper_1804_10694_b200/_lib/libtm.so} timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-product}', '$c', d['step_ms']['median'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
  done
done
done

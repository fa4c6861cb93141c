# EXPERIMENT: one lane per warp polls the split's and epilogue's mbarriers (TM_DC_EXP=7)
# vs every lane; conv parity through the experiment library, then interleaved timing.
TM_LIB_PATH=_exp/libtm_poll1.so timeout 300 python -m pytest tests/test_conv.py -q -x -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do
  for v in product poll1; do
    L=; [ $v != product ] && L=_exp/libtm_$v.so
    env ${L:+TM_LIB_PATH=$L} bash scripts/ms.sh "conv3 $v" --config CONV --steps 20 --warmup 5 --no-cpu
    env ${L:+TM_LIB_PATH=$L} bash scripts/ms.sh "conv5 $v" --config CONV --conv-r 5 --steps 20 --warmup 5 --no-cpu
    env ${L:+TM_LIB_PATH=$L} bash scripts/ms.sh "conv9 $v" --config CONV --conv-r 9 --steps 10 --warmup 3 --no-cpu
  done
done

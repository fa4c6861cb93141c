# EXPERIMENT (conv, timing + parity through the product tests): TMEM store shape (x16: two
# 16-column stores per stage instead of one x32) and A-slot placement (tend: A slots at the
# top of TMEM instead of right after the accumulators).  Interleaved, one box.
for i in 1 2; do
  for v in product x16 tend; do
    L=; [ $v != product ] && L=_exp/libtm_$v.so
    env ${L:+TM_LIB_PATH=$L} bash scripts/ms.sh "conv3 $v" --config CONV --steps 20 --warmup 5 --no-cpu
    env ${L:+TM_LIB_PATH=$L} bash scripts/ms.sh "conv5 $v" --config CONV --conv-r 5 --steps 20 --warmup 5 --no-cpu
  done
done

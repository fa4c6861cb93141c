# EXPERIMENT (timing only, wrong results): which role bounds the direct conv after the
# two-row tiles.  x1: A_hi*B_lo MMA dropped; x2: split's TMEM stores dropped; x3: epilogue's
# TMEM loads dropped.  Interleaved runs on one box.
for i in 1 2; do
  bash scripts/ms.sh "conv3 base" --config CONV --steps 20 --warmup 5 --no-cpu
  for x in x1 x2 x3; do TM_LIB_PATH=_exp/libtm_$x.so bash scripts/ms.sh "conv3 $x" --config CONV --steps 20 --warmup 5 --no-cpu; done
done
bash scripts/ms.sh "conv5 base" --config CONV --conv-r 5 --steps 20 --warmup 5 --no-cpu
for x in x1 x2 x3; do TM_LIB_PATH=_exp/libtm_$x.so bash scripts/ms.sh "conv5 $x" --config CONV --conv-r 5 --steps 20 --warmup 5 --no-cpu; done

# NOTE: the noalo libraries this compared were built from tc_gemm_nn.cu alone, which
# DESIGN 7.15 shows can silently keep the product kernels -- results inconclusive, not used.
# EXPERIMENT: A_lo staged in TMEM (tcgen05.st, the shipped rule) vs in shared memory
# (noalo2: 2 lo stages, noalo4: 4 lo stages for stages <= 20 KiB) on C4 / C2 / C3;
# 1xTF32 (no split) as the streaming floor of the same pipeline.  Interleaved, one box.
for i in 1 2; do
  for c in C4 C2; do
    bash scripts/ms.sh "$c base" --config $c --steps 50 --warmup 5 --no-cpu --no-e2e
    for x in noalo2 noalo4; do TM_LIB_PATH=_exp/libtm_$x.so bash scripts/ms.sh "$c $x" --config $c --steps 50 --warmup 5 --no-cpu --no-e2e; done
  done
done
bash scripts/ms.sh "C4 tf32x1" --config C4 --algo tf32x1 --steps 50 --warmup 5 --no-cpu --no-e2e
for x in base noalo4; do
  if [ $x = base ]; then L=; else L=_exp/libtm_$x.so; fi
  env ${L:+TM_LIB_PATH=$L} bash scripts/ms.sh "C3 $x" --config C3 --steps 10 --warmup 3 --no-cpu --no-e2e
done

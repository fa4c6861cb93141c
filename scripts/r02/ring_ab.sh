# EXPERIMENT: ring depths (r02_exp_macros-style knobs TM_EXP_LO_CAP / TM_EXP_BUDGET_KB, all six
# tc_gemm.cuh TUs rebuilt): lo4 = lo ring <= 4, 204 KiB budget (C4: 9 raw stages); lo2 = lo ring 2.
for i in 1 2; do
  for v in product lo4 lo2; do
    L=; [ $v != product ] && L=_exp/libtm_$v.so
    for c in C4 C2; do env ${L:+TM_LIB_PATH=$L} bash scripts/ms.sh "$c $v" --config $c --steps 50 --warmup 5 --no-cpu --no-e2e; done
    env ${L:+TM_LIB_PATH=$L} bash scripts/ms.sh "C3 $v" --config C3 --steps 20 --warmup 5 --no-cpu --no-e2e
  done
done

# EXPERIMENT (temporary knob, timing only): drop the A_hi*B_lo MMA after the truncated-lo split change
for i in 1 2; do bash scripts/ms.sh "conv" --config CONV --steps 20 --warmup 5 --no-cpu; TM_DC_EXP_SKIP=1 bash scripts/ms.sh "conv skip-1-mma" --config CONV --steps 20 --warmup 5 --no-cpu; done

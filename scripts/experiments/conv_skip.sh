# NOTE: TM_DC_EXP_SKIP was a temporary knob of the experiment build (not in the library); results in DESIGN.md 6.4
# EXPERIMENT (timing only, wrong results): which role bounds the direct conv
bash scripts/ms.sh "conv" --config CONV --steps 20 --warmup 5 --no-cpu
for x in 1 2 4 6 7; do TM_DC_EXP_SKIP=$x bash scripts/ms.sh "conv skip=$x" --config CONV --steps 20 --warmup 5 --no-cpu; done

for sl in 2 4 6 8; do TM_DC_SLOTS=$sl bash scripts/ms.sh "conv slots=$sl" --config CONV --steps 20 --warmup 5 --no-cpu; done
TM_DC_SLOTS=6 bash scripts/ms.sh "conv slots=6 beta.5" --config CONV --conv-beta 0.5 --steps 20 --warmup 5 --no-cpu
bash scripts/ms.sh "conv slots=4 beta.5" --config CONV --conv-beta 0.5 --steps 20 --warmup 5 --no-cpu

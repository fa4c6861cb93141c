for c in C4 C2; do
bash scripts/ms.sh "$c default" --config $c --steps 30 --warmup 5 --no-cpu --no-e2e
TM_COOPERATIVE=0 bash scripts/ms.sh "$c coop=0" --config $c --steps 30 --warmup 5 --no-cpu --no-e2e
TM_TC_CONFIG=2,32,0 bash scripts/ms.sh "$c 2,32,0" --config $c --steps 30 --warmup 5 --no-cpu --no-e2e
TM_TC_CONFIG=2,64,0 bash scripts/ms.sh "$c 2,64,0" --config $c --steps 30 --warmup 5 --no-cpu --no-e2e
TM_TC_CONFIG=1,64,0 bash scripts/ms.sh "$c 1,64,0" --config $c --steps 30 --warmup 5 --no-cpu --no-e2e
done

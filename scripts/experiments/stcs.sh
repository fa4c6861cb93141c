# EXPERIMENT: streaming (evict-first) float4 stores in the epilogue
for c in C4 C2; do bash scripts/ms.sh "$c" --config $c --steps 30 --warmup 5 --no-cpu --no-e2e; done
bash scripts/ms.sh "conv" --config CONV --steps 20 --warmup 5 --no-cpu
bash scripts/ms.sh "conv beta.5" --config CONV --conv-beta 0.5 --steps 20 --warmup 5 --no-cpu
bash scripts/ms.sh "C5" --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e

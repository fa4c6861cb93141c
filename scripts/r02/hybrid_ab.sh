# A/B of the stream-K schedule: TM_SK_HYBRID=0 (pure stream-K), 1 (partial wave only,
# then whole tiles), 2 (partial wave + one full wave) on the shapes whose plan is stream-K.
for i in 1 2; do
  for h in 0 1 2; do
    for c in C4 C3; do TM_SK_HYBRID=$h bash scripts/ms.sh "$c hybrid=$h" --config $c --steps 30 --warmup 5 --no-cpu --no-e2e; done
    TM_SK_HYBRID=$h bash scripts/ms.sh "C3b tf32x1 hybrid=$h" --config C3b --algo tf32x1 --steps 10 --warmup 3 --no-cpu --no-e2e
  done
done

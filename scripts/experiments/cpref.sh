# NOTE: TM_C_PREFETCH was a temporary knob of the experiment build (not in the library); result in DESIGN.md 6.1
for c in C2 C4 C1; do for pf in 1 0; do TM_C_PREFETCH=$pf bash scripts/ms.sh "$c prefetch=$pf" --config $c --steps 30 --warmup 5 --no-cpu --no-e2e; done; done
rm -f /tmp/t.jsonl
S=1060 python scripts/experiments/epi_probe.py; mv gpurun_out/trace_epi_b0.5.jsonl gpurun_out/trace_pf1.jsonl
TM_C_PREFETCH=0 S=1060 python scripts/experiments/epi_probe.py; mv gpurun_out/trace_epi_b0.5.jsonl gpurun_out/trace_pf0.jsonl

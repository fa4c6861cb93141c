# C1/C2 latency breakdown: event-timed configs, per-CTA %globaltimer traces, ncu full of C2 and C1.
set -u
python scripts/r02/latency_probe.py 2>&1 | tee gpurun_out/latency_probe_r02.txt
rm -f /tmp/tr.jsonl
python scripts/r02/trace_c2.py /tmp/tr.jsonl 2,64,1/0.5 2,64,0/0.5 1,128,1/0.5 1,64,1/0.5 1,128,0/0.5
python scripts/trace_report.py /tmp/tr.jsonl > gpurun_out/trace_c2_r02.txt 2>&1
for c in C1 C2 C4; do
  TM_COOPERATIVE=0 timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_sgemm -s 3 -c 1 -o gpurun_out/prof_${c}_r02 python bench.py --config $c --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
ls gpurun_out

# Round-2 full GPU pass: smoke, all GPU tests, default bench line, per-config lines
# (C1-C5, C3b variants, CONV 3x3..11x11 and the paper-exact valid shape, BLUR),
# the reference arm, a launch list of the default bench and ncu --set full captures
# of the dominant kernel of each config.
set -u
TAG=${TAG:-r02}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests/ -m gpu -q -p no:cacheprovider --timeout 600 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err; tail -1 gpurun_out/bench_default_$TAG.json | cut -c1-300
{
for c in C1 C2 C3 C3b C4; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1; done
timeout 300 python bench.py --config C3 --algo simt --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1
timeout 300 python bench.py --config C3b --algo tf32x1 --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1
timeout 300 python bench.py --config C3b --algo bf16x9 --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1
for r in 3 5 7 9 11; do timeout 300 python bench.py --config CONV --conv-r $r --steps 20 --warmup 5 --no-cpu 2>/dev/null | tail -1; done
timeout 300 python bench.py --config CONV --conv-valid --steps 20 --warmup 5 --no-cpu 2>/dev/null | tail -1
timeout 300 python bench.py --config CONV --conv-beta 0.5 --steps 20 --warmup 5 --no-cpu 2>/dev/null | tail -1
timeout 300 python bench.py --config BLUR --steps 50 --warmup 5 2>/dev/null | tail -1
} > gpurun_out/bench_configs_$TAG.jsonl
cut -c1-160 gpurun_out/bench_configs_$TAG.jsonl
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_$TAG.json 2>&1; tail -1 gpurun_out/bench_reference_$TAG.json | cut -c1-200
TM_COOPERATIVE=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
for c in C5 C4 C3 C2; do
  TM_COOPERATIVE=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sgemm_tc -s 3 -c 1 -o gpurun_out/prof_${c}_$TAG python bench.py --config $c --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_sgemm_small -s 3 -c 1 -o gpurun_out/prof_C1_$TAG python bench.py --config C1 --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
TM_COOPERATIVE=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sgemm_simt -s 2 -c 1 -o gpurun_out/prof_simt_c3_$TAG python bench.py --config C3 --algo simt --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_direct -s 1 -c 1 -o gpurun_out/prof_conv_$TAG python bench.py --config CONV --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_blur -s 3 -c 1 -o gpurun_out/prof_blur_$TAG python bench.py --config BLUR --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
ls gpurun_out | grep $TAG
# summaries on the box (the reports together exceed gpurun's 64 MiB return limit)
for f in gpurun_out/prof_*_$TAG.ncu-rep; do
  b=$(basename $f .ncu-rep)
  python scripts/ncu_summary.py $f > gpurun_out/ncu_${b#prof_}.txt 2>&1
done
python scripts/ncu_summary.py --launches gpurun_out/launches_c5_$TAG.csv > gpurun_out/launches_c5_$TAG.txt 2>&1
mkdir -p gpurun_out/keep && mv gpurun_out/prof_C2_$TAG.ncu-rep gpurun_out/prof_blur_$TAG.ncu-rep gpurun_out/keep/ 2>/dev/null
rm -f gpurun_out/prof_*_$TAG.ncu-rep
du -sh gpurun_out

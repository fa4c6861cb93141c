set -x
ncu --set full --clock-control none --import-source on -k regex:k_sgemm_tc -s 2 -c 1 -o gpurun_out/prof_c3b_r01 python bench.py --config C3b --steps 2 --warmup 2 --no-cpu --no-e2e > gpurun_out/ncu_c3b.log 2>&1
tail -3 gpurun_out/ncu_c3b.log
ncu --set full --clock-control none --import-source on -k regex:k_sgemm_tc -s 1 -c 1 -o gpurun_out/prof_c5_r01 python bench.py --config C5 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_c5.log 2>&1
tail -3 gpurun_out/ncu_c5.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_r01.csv python bench.py --steps 3 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
ls -la gpurun_out

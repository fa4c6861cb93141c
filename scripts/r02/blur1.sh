# Blur: parity tests, bench line, launch list and one ncu --set full capture of k_blur.
set -u
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_blur.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -15
timeout 300 python bench.py --config BLUR --steps 50 --warmup 5 2>&1 | tail -1 > gpurun_out/bench_blur_r02.json
cut -c1-900 gpurun_out/bench_blur_r02.json
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_blur -s 3 -c 1 -o gpurun_out/prof_blur_r02 python bench.py --config BLUR --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_blur_r02.csv python bench.py --config BLUR --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1
grep k_blur gpurun_out/launches_blur_r02.csv | head -6

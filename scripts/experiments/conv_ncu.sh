ncu --set full --clock-control none --import-source on -k regex:k_conv_direct -s 1 -c 1 -o gpurun_out/prof_conv_ring python bench.py --config CONV --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ls -la gpurun_out

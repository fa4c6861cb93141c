TM_DC_LY=1 ncu --set full --clock-control none --import-source on -k regex:k_conv_direct -s 1 -c 1 -o gpurun_out/prof_conv_ring_ly1 python bench.py --config CONV --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
TM_DC_LY=16 ncu --set full --clock-control none --import-source on -k regex:k_conv_direct -s 1 -c 1 -o gpurun_out/prof_conv_ring_ly16 python bench.py --config CONV --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ls gpurun_out/*.ncu-rep

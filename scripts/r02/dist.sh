set -u
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_dist_loopback.py tests/test_dist_nccl.py -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -5
timeout 900 python scripts/scaling_projection.py 2>&1 | tail -1 > gpurun_out/scaling_projection_r02.json; cat gpurun_out/scaling_projection_r02.json

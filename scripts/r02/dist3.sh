set -u
timeout 900 python -m pytest tests/test_dist_loopback.py tests/test_dist_nccl.py tests/test_dist_gloo.py -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -3
for p in 8 4 2; do P=$p python scripts/r02/dist_probe.py; done
timeout 900 python scripts/scaling_projection.py 2>&1 | tail -4
TM_DIST_CHUNKS=uniform timeout 900 python scripts/scaling_projection.py 2>&1 | tail -4 | head -3

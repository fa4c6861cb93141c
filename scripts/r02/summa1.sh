set -u
timeout 900 python -m pytest tests/test_summa.py tests/test_dist_nccl.py tests/test_bench_contract.py -q -p no:cacheprovider --timeout 600 2>&1 | tail -15

set -u
timeout 900 python -m pytest tests/test_dist_ce.py -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -15

set -u
timeout 600 python -m pytest tests/test_blur.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -3
python scripts/r02/blur_probe.py

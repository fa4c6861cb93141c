# row-ring conv variant with per-block (not per-tile) tile decoding
timeout 600 python -m pytest tests/test_conv.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -2
for ly in 1 8 16 32; do TM_DC_LY=$ly bash scripts/ms.sh "conv ring ly=$ly" --config CONV --steps 20 --warmup 5 --no-cpu; done

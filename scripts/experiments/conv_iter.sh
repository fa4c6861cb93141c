# NOTE: TM_DC_LY / TM_DC_ROWS belong to the row-ring variant in conv_row_ring.patch (not adopted)
timeout 600 python -m pytest tests/test_conv.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -2
for i in 1 2; do bash scripts/ms.sh "conv" --config CONV --steps 20 --warmup 5 --no-cpu; done
bash scripts/ms.sh "conv beta.5" --config CONV --conv-beta 0.5 --steps 20 --warmup 5 --no-cpu

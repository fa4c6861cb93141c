timeout 600 python -m pytest tests/test_conv.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -3
bash scripts/ms.sh "conv old" --config CONV --steps 20 --warmup 5 --no-cpu
TM_DC_ROWBOX=1 bash scripts/ms.sh "conv old rowboxes" --config CONV --steps 20 --warmup 5 --no-cpu
TM_DC_ROWBOX=1 timeout 600 python -m pytest tests/test_conv.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -3

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import torch;print(torch.cuda.get_device_name(0))"
timeout 300 python -m pytest tests/test_probes.py -x -q -p no:cacheprovider 2>&1 | tail -30
cat gpurun_out/probes.json
timeout 900 python -m pytest tests/test_parity.py -q -p no:cacheprovider --timeout 300 2>&1 | tail -60

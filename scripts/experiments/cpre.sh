# NOTE: measured with a temporary build that preloaded beta*C during the last K_c chunk (reverted); DESIGN.md 6.1
timeout 600 python -m pytest tests/test_parity.py tests/test_transposes.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -2
for c in C2 C4 C1 C2 C4; do bash scripts/ms.sh "$c" --config $c --steps 30 --warmup 5 --no-cpu --no-e2e; done
S=1060 python scripts/experiments/epi_probe.py

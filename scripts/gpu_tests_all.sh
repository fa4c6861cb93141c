python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1200 python -m pytest tests/ -m gpu -q -p no:cacheprovider --timeout 300 --durations=8 2>&1 | tail -25

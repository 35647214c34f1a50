# full GPU test suite (what the driver runs at round end), with a time limit
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -25

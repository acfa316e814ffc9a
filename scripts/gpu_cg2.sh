set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cfg1" 2>&1 | tail -30
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -30

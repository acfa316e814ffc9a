set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 120 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "quantize or pack_weights" 2>&1 | tail -20
timeout 120 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cfg1" 2>&1 | tail -40
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q 2>&1 | tail -60

set -x
NVCC_APPEND_FLAGS="-DCONVQ_HANG_CHECK" python paper_2202_06819_b200/_build.py --force
for bo in 1 0; do
CONV_Q_DESC_BO=$bo timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cfg1 or edge" 2>&1 | tail -12
done

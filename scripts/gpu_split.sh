set -x
export NVCC_APPEND_FLAGS="-DCONVQ_HANG_CHECK"
python paper_2202_06819_b200/_build.py > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "split or cfg1" 2>&1 | tail -5
unset NVCC_APPEND_FLAGS
python paper_2202_06819_b200/_build.py > /dev/null 2>&1
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
TRACE_NET=resnet18 TRACE_N=1 TRACE_BITS=8 timeout 200 python scripts/trace.py l4.b1.c2 2>&1 | sort -k2 -n | head -8
timeout 400 python bench.py --workload resnet18_int8_b1 --no-cpu-baseline --no-k7 --no-stem > gpurun_out/b18.json 2> gpurun_out/b18.err; head -c 400 gpurun_out/b18.json; grep -E "^  l" gpurun_out/b18.err
timeout 400 python bench.py --workload resnet18_int4_b16 --no-cpu-baseline --no-k7 --no-stem > gpurun_out/b18i4.json 2> gpurun_out/b18i4.err; head -c 400 gpurun_out/b18i4.json; grep -E "^  l" gpurun_out/b18i4.err

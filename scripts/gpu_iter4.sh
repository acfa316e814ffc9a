set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -5
timeout 600 python bench.py --no-cpu-baseline --layers-out gpurun_out/layers_r50_int8.json > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err
cat gpurun_out/bench_r50.json; cat gpurun_out/bench_r50.err

#!/bin/bash
# parity (pytest -m gpu) + default bench with per-layer table; outputs under gpurun_out/
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? ; tail -3 gpurun_out/pytest_gpu.log
python bench.py --layers-out gpurun_out/layers.json ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cat gpurun_out/bench.json

#!/bin/bash
# default bench (as the driver runs it) with the per-layer table; outputs under gpurun_out/
python bench.py --layers-out gpurun_out/layers.json ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cat gpurun_out/bench.json

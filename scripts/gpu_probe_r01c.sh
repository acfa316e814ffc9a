#!/bin/bash
# micro-probes + per-CTA traces of the epilogue-bound layers (round 1, session 2)
cd scripts/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_rates pipe_rates.cu && ./pipe_rates > ../../gpurun_out/pipe_rates.txt 2>&1; cd ../..
for l in l1.b0.c3 l3.b1.c3 l4.b1.c3 l1.b0.c2 l2.b1.c3; do
  timeout 120 python scripts/trace.py $l >> gpurun_out/trace_r01c.txt 2>&1
done

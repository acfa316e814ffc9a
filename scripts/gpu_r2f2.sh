#!/bin/bash
# round 2: TMA-loaded residual skip slabs -- residual parity (every candidate), full suite, residual bench + candidate times
O=gpurun_out/r2f2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_network.py tests/test_gpu_unsigned.py -q -x -rf -k "residual or unsigned" > $O/res_tests.log 2>&1; echo "rc=$?" >> $O/res_tests.log
timeout 1800 python -m pytest tests -m gpu -q -rf > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
for l in l1.b0.c3 l3.b1.c3; do timeout 300 python scripts/res_cands.py $l 256 > $O/res_$l.txt 2>&1; done
CONV_Q_CACHE=$O/cache_res.json timeout 900 python bench.py --workload resnet50_int8_b256_res --steps 50 --warmup 5 --no-cpu-baseline --no-k7 --layers-out $O/layers_res.json > $O/bench_res.json 2> $O/bench_res.err
tail -2 $O/res_tests.log; tail -2 $O/gputest.log

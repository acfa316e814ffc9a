#!/bin/bash
# round 2: runtime pipeline depth (WS region sized to the layer) -- parity suite + bench
O=gpurun_out/r2d; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x -rf > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
CONV_Q_CACHE=$O/cache_r50.json timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --layers-out $O/layers_r50.json > $O/bench_r50.json 2> $O/bench_r50.err
CONV_Q_CACHE=$O/cache_r50_uns.json timeout 900 python bench.py --workload resnet50_int8_b256_uns --steps 50 --warmup 5 --no-cpu-baseline --no-k7 --layers-out $O/layers_r50_uns.json > $O/bench_r50_uns.json 2> $O/bench_r50_uns.err
tail -3 $O/gputest.log

#!/bin/bash
# round 2: graph-timed tuning -- tuning tests, b1 / INT4 b16 / b256 benches re-tuned, probe modes (graph-timed)
O=gpurun_out/r2g; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -rf -k "tune or tuned or bench_chain or every_candidate" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for w in resnet18_int8_b1 resnet18_int4_b16 resnet50_int8_b256; do
  CONV_Q_CACHE=$O/cache_$w.json timeout 900 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --no-k7 --layers-out $O/layers_$w.json > $O/bench_$w.json 2> $O/bench_$w.err
done
PROBE_CFG=bm256_bn256_kc128x1_c2,bm256_bn128_kc128x2_c2_st,bm256_bn256_kc128x2_c2_st,bm128_bn256_kc128x1_c1,bm128_bn128_kc128x2_c1_w,bm128_bn256_kc128x2_c1_w,bm256_bn128_kc128x3_c2_st_h timeout 600 python scripts/probe.py l4.b1.c1 l3.b1.c2 l3.b1.c3 > $O/probe.txt 2>&1
tail -2 $O/tests.log

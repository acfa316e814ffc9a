#!/bin/bash
# round-2 evidence for the current build: full GPU suite + smoke, every workload's bench line
O=gpurun_out/fin; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rf > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
CONV_Q_CACHE=$O/cache_r50.json timeout 900 python bench.py --steps 20 --warmup 5 --layers-out $O/layers_resnet50_int8_b256.json > $O/bench_resnet50_int8_b256.json 2> $O/bench_resnet50_int8_b256.err
for w in resnet50_int8_b256_res resnet50_int8_b256_uns resnet18_int4_b16 resnet18_int8_b1 resnet18_int4_b16_uns; do
  CONV_Q_CACHE=$O/cache_$w.json timeout 900 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --no-k7 --layers-out $O/layers_$w.json > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
tail -3 $O/gputest.log

#!/bin/bash
# residual epilogue with FADD2 skip conversion: GPU suite + residual bench A/B vs the previous build
O=gpurun_out/r2ah; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
tail -3 $O/gputest.log
REF=$PWD/paper_2202_06819_b200/libconvq_ref.so
for i in 1 2; do for v in new ref; do
  if [ $v = ref ]; then export CONV_Q_LIB=$REF; else unset CONV_Q_LIB; fi
  timeout 600 python bench.py --workload resnet50_int8_b256_res --steps 50 --warmup 5 --no-cpu-baseline --no-k7 --no-e2e > $O/bench_${v}_$i.json 2> $O/bench_${v}_$i.err
done; done
unset CONV_Q_LIB
for f in $O/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['parity_ok'], d.get('graph_layers_sum_ms'))"; done

#!/bin/bash
# late accumulator commit (libconvq_la.so) vs default: parity + candidate times + bench A/B
O=gpurun_out/r2ag; mkdir -p $O
LA=$PWD/paper_2202_06819_b200/libconvq_la.so
CONV_Q_LIB=$LA timeout 1500 python -m pytest tests -m gpu -q -rf -x > $O/gputest_la.log 2>&1; echo "rc=$?" >> $O/gputest_la.log
tail -3 $O/gputest_la.log
for v in la def; do
  if [ $v = la ]; then export CONV_Q_LIB=$LA; else unset CONV_Q_LIB; fi
  CT_TOP=2 timeout 600 python scripts/cand_times.py 256 l3.b1.c3 l2.b1.c3 l3.b1.c1 l4.b1.c3 l4.b1.c1 l3.b1.c2 l2.b1.c2 > $O/cand_$v.txt 2>&1
done
for i in 1 2; do for v in la def; do
  if [ $v = la ]; then export CONV_Q_LIB=$LA; else unset CONV_Q_LIB; fi
  timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-k7 --no-e2e > $O/bench_${v}_$i.json 2> $O/bench_${v}_$i.err
done; done
unset CONV_Q_LIB
paste $O/cand_la.txt $O/cand_def.txt
for f in $O/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['parity_ok'], d.get('graph_layers_sum_ms'))"; done

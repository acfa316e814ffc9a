#!/bin/bash
# INT4 with 4 epilogue warpgroups (libconvq_wgi44.so) vs 2 (libconvq.so): INT4 parity + candidate times + bench
O=gpurun_out/r2t; mkdir -p $O
V=$PWD/paper_2202_06819_b200/libconvq_wgi44.so
CONV_Q_LIB=$V timeout 1500 python -m pytest tests -m gpu -q -rf > $O/gputest_wg4.log 2>&1; echo "rc=$?" >> $O/gputest_wg4.log
tail -3 $O/gputest_wg4.log
for v in wg4 wg2; do
  if [ $v = wg4 ]; then export CONV_Q_LIB=$V; else unset CONV_Q_LIB; fi
  CT_BITS=4 CT_TOP=3 timeout 600 python scripts/cand_times.py 256 l1.b0.c3 l1.b1.c1 l1.b0.c2 l2.b1.c3 l3.b1.c3 l3.b1.c2 l4.b1.c1 l4.b1.c3 > $O/cand4_$v.txt 2>&1
  CT_BITS=4 CT_TOP=3 CT_NET=resnet18 timeout 600 python scripts/cand_times.py 16 l1.b0.c1 l2.b1.c1 l3.b1.c1 l4.b1.c1 > $O/cand4r18_$v.txt 2>&1
  for w in resnet18_int4_b16 resnet18_int4_b16_uns; do
    timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --no-k7 --no-e2e > $O/bench_${w}_$v.json 2> $O/bench_${w}_$v.err
  done
done
unset CONV_Q_LIB
paste $O/cand4_wg4.txt $O/cand4_wg2.txt; paste $O/cand4r18_wg4.txt $O/cand4r18_wg2.txt
for f in $O/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['parity_ok'])"; done

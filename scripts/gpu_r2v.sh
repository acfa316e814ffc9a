#!/bin/bash
# INT4 ReLU epilogue without shift / min: parity (full suite) + A/B vs the previous build (libconvq_ref.so)
O=gpurun_out/r2v; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
tail -3 $O/gputest.log
REF=$PWD/paper_2202_06819_b200/libconvq_ref.so
for v in new ref; do
  if [ $v = ref ]; then export CONV_Q_LIB=$REF; else unset CONV_Q_LIB; fi
  CT_BITS=4 CT_TOP=2 timeout 600 python scripts/cand_times.py 256 l1.b0.c3 l1.b1.c1 l1.b0.c2 l2.b1.c3 l3.b1.c3 l3.b1.c2 l4.b1.c1 l4.b1.c3 > $O/cand4_$v.txt 2>&1
  CT_BITS=4 CT_TOP=2 CT_NET=resnet18 timeout 600 python scripts/cand_times.py 16 l1.b0.c1 l2.b1.c1 l3.b1.c1 l4.b1.c1 > $O/cand4r18_$v.txt 2>&1
  for w in resnet18_int4_b16 resnet18_int4_b16_uns; do
    timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --no-k7 --no-e2e > $O/bench_${w}_$v.json 2> $O/bench_${w}_$v.err
  done
done
unset CONV_Q_LIB
paste $O/cand4_new.txt $O/cand4_ref.txt; paste $O/cand4r18_new.txt $O/cand4r18_ref.txt
for f in $O/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['parity_ok'])"; done

#!/bin/bash
# magic s32->f32 epilogue conversion: full GPU suite, candidate-time A/B, bench A/B
O=gpurun_out/r2q; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
tail -4 $O/gputest.log
for nm in 1 0; do
  CONV_Q_NO_MAGIC=$nm timeout 400 python scripts/cand_times.py 256 l3.b1.c3 l1.b0.c3 l1.b1.c1 l2.b1.c3 l1.b0.c1 l2.b0.c1 > $O/cand_nm$nm.txt 2>&1
done
for i in 1 2; do
for nm in 1 0; do
  CONV_Q_NO_MAGIC=$nm timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-k7 --no-e2e --layers-out $O/layers_nm${nm}_$i.json > $O/bench_nm${nm}_$i.json 2> $O/bench_nm${nm}_$i.err
done; done
paste $O/cand_nm1.txt $O/cand_nm0.txt | head -80
for f in $O/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['frac'], d['parity_ok'], d.get('graph_layers_sum_ms'))"; done

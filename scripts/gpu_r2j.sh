#!/bin/bash
# round 2: epilogue-released last stage -- parity, candidate times A/B, bench A/B
O=gpurun_out/r2j; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
for er in 1 0; do
  CONV_Q_EPI_RELEASE=$er timeout 400 python scripts/cand_times.py 256 l3.b1.c3 l2.b1.c3 l1.b0.c3 l4.b1.c1 > $O/cand_er$er.txt 2>&1
  CONV_Q_EPI_RELEASE=$er CONV_Q_CACHE=$O/cache_er$er.json timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-k7 --no-e2e --layers-out $O/layers_er$er.json > $O/bench_er$er.json 2> $O/bench_er$er.err
done
tail -2 $O/gputest.log

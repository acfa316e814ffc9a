#!/bin/bash
# NEXT-4 follow-up: search tests, bench A/B exhaustive tuning vs learned search (twice each, alternating)
O=gpurun_out/r2m; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_search.py -q -rf > $O/gputest_search.log 2>&1; echo "rc=$?" >> $O/gputest_search.log
tail -3 $O/gputest_search.log
for i in 1 2; do
  timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-k7 --no-e2e --layers-out $O/layers_ex$i.json > $O/bench_ex$i.json 2> $O/bench_ex$i.err
  timeout 1200 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-k7 --no-e2e --search 128 --layers-out $O/layers_se$i.json > $O/bench_se$i.json 2> $O/bench_se$i.err
done
for f in $O/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['frac'], d['parity_ok'], d.get('tuning'))"; done

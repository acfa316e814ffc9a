#!/bin/bash
# round 2 (session 3): re-validate HEAD -- GPU suite + smoke + default bench
O=gpurun_out/r2k; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
CONV_Q_CACHE=$O/cache_r50.json timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --layers-out $O/layers_r50.json > $O/bench_r50.json 2> $O/bench_r50.err
timeout 2400 python -m pytest tests -m gpu -q -rf > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
tail -3 $O/gputest.log; cat $O/bench_r50.json

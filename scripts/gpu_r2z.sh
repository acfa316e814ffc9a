#!/bin/bash
# final verification of HEAD, the way the driver runs it: GPU suite, smoke, default bench, reference arm
O=gpurun_out/r2z; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 --layers-out $O/layers_r50.json > $O/bench_r50.json 2> $O/bench_r50.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
tail -2 $O/gputest.log; cat $O/smoke.log; tail -1 $O/bench_r50.json | cut -c1-600; tail -1 $O/bench_reference.json | cut -c1-300

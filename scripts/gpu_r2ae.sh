#!/bin/bash
# s8 C = 16 (mod 32) ragged channel blocks: full GPU suite (new parity cases) + bench sanity
O=gpurun_out/r2ae; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -rf -k ragged > $O/ragged.log 2>&1; echo "rc=$?" >> $O/ragged.log
tail -3 $O/ragged.log
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
tail -3 $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log; cat $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_r50.json 2> $O/bench_r50.err
python -c "import json; d=json.loads(open('$O/bench_r50.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['parity_ok'], d['e2e']['value'])"

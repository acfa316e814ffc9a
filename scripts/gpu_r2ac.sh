#!/bin/bash
# flakiness check: the GPU suite three times in a row, plus the default bench twice
O=gpurun_out/r2ac; mkdir -p $O
for i in 1 2 3; do
  timeout 1500 python -m pytest tests -m gpu -q -rf -p no:randomly > $O/gputest_$i.log 2>&1; echo "rc=$?" >> $O/gputest_$i.log
  tail -2 $O/gputest_$i.log
done

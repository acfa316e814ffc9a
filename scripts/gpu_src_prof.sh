#!/bin/bash
# ncu --set full with source-level stall sampling for a few layers (args: layer[:config] ...)
for lc in "$@"; do
  l=${lc%%:*}; c=""; [[ "$lc" == *:* ]] && c="--config ${lc#*:}"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 -o gpurun_out/src_$l \
    python scripts/prof_layer.py --layer $l $c > gpurun_out/src_$l.log 2>&1
  tail -1 gpurun_out/src_$l.log
done

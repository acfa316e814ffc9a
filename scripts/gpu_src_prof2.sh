#!/bin/bash
# ncu source-level profile of one layer/config in a probe mode: args layer config probe tag
l=$1; c=$2; m=$3; tag=$4
CONV_Q_PROBE=$m timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 -o gpurun_out/src_$tag \
    python scripts/prof_layer.py --layer $l --config $c > gpurun_out/src_$tag.log 2>&1
tail -1 gpurun_out/src_$tag.log

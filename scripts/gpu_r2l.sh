#!/bin/bash
# NEXT-4: device parity of the enlarged space + search; Table 1 analog and ResNet-50 layers
O=gpurun_out/r2l; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_search.py -q -rf > $O/gputest_search.log 2>&1; echo "rc=$?" >> $O/gputest_search.log
tail -3 $O/gputest_search.log
timeout 1500 python scripts/search_table1.py $O/search_table1.json 128 8,4 l3.b1.c3@256 l4.b1.c1@256 l4.b1.c3@256 l1.b0.c3@256 l3.b1.c2@256 l2.b1.c3@256 > $O/search_table1.log 2>&1; echo "rc=$?" >> $O/search_table1.log
tail -30 $O/search_table1.log

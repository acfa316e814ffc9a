#!/bin/bash
# ncu --set full of INT4 layers (l1.b0.c3 and l3.b1.c3 at b256) with source-level stall attribution
O=gpurun_out/r2u2; mkdir -p $O
for l in l1.b0.c3 l3.b1.c3; do
  c=$(CT_BITS=4 CT_TOP=1 python scripts/cand_times.py 256 $l 2>/dev/null | sed -n 2p | awk '{print $1}')
  echo "$l $c"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 -o $O/full4_$l \
    python scripts/prof_layer.py --layer $l --bits 4 --config $c > $O/full4_$l.log 2>&1
  python scripts/ncu_summary.py $O/full4_$l.ncu-rep > $O/r02s3b_full_int4_$l.txt 2>&1
done
python scripts/ncu_src_top.py $O/full4_l1.b0.c3.ncu-rep $((256*56*56*256)) > $O/r02s3b_src_int4_l1.b0.c3.txt 2>&1
rm -f $O/*.ncu-rep
cat $O/r02s3b_full_int4_*.txt | head -80; head -40 $O/r02s3b_src_int4_l1.b0.c3.txt

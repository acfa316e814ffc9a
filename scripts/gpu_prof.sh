set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 -o gpurun_out/prof_l1c3 python scripts/prof_layer.py --layer l1.b0.c3 --config bm128_bn128_kc64x4_c1 > gpurun_out/ncu_l1c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 -o gpurun_out/prof_l3c2 python scripts/prof_layer.py --layer l3.b1.c2 --config bm128_bn256_kc128x1_c1_st > gpurun_out/ncu_l3c2.log 2>&1
tail -3 gpurun_out/ncu_l1c3.log gpurun_out/ncu_l3c2.log

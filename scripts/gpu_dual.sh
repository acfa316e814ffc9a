# dual-MMA build: the previously failing configs at N=256, full parity suite, then the bench
export CONV_Q_LIB=$PWD/paper_2202_06819_b200/libconvq_dual.so
for c in bm128_bn64_kc128x2_c1 bm128_bn64_kc128x2_c1_w; do for i in 1 2 3; do timeout 60 python scripts/check_cfg.py l1.b1.c1 $c 256 2>&1 | tail -1; done; done
timeout 60 python scripts/check_cfg.py l2.b0.c1 bm128_bn64_kc128x2_c1_w 256 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --no-cpu-baseline --no-k7 --layers-out gpurun_out/layers_dual.json > gpurun_out/bench_dual.json 2> gpurun_out/bench_dual.err; echo bench=$?; head -c 300 gpurun_out/bench_dual.json

timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for n in 8 256; do timeout 60 python scripts/check_cfg.py l1.b0.c2 bm256_bn64_kc64x1_c2_st_h_w_m2 $n 2>&1 | tail -1; done
timeout 300 python scripts/stem_probe.py 256 8 2>&1 | grep -E "_h_w|tuned|total"
export PROBE_CFG=bm128_bn64_kc64x1_c1_st_h_w_m2,bm256_bn64_kc64x1_c2_st_h_w,bm256_bn64_kc64x1_c2_st_h_w_m2
export PROBE_MODES=0
timeout 300 python scripts/probe.py l1.b0.c2

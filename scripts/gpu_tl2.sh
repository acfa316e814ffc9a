for w in "0 0" "2 100" "2 400" "1 100000"; do
  set -- $w
  echo "##### EPI_WAIT=$1 NS=$2"
  for lc in "l1.b0.c2 bm128_bn64_kc64x1_c1_st_h_w" "stem bm128_bn64_kc64x1_c1_st_h_w" "l1.b0.c1 bm128_bn64_kc64x1_c1_w"; do
    set -- $lc
    for m in 0 7; do echo "=== $1 probe $m"; CONV_Q_EPI_WAIT=${w% *} CONV_Q_EPI_WAIT_NS=${w#* } CONV_Q_PROBE=$m timeout 120 python scripts/timeline.py $1 $2 256 10 2>&1 | grep "MMA commit"; done
  done
done

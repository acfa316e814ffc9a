# launch list + full captures with the tile picks of the timed bench (scratch/tune_r50.json)
export CONV_Q_CACHE=$PWD/scratch/tune_r50.json
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r01_launches.csv python bench.py --no-tune --steps 2 --warmup 3 --no-e2e --no-stem --no-cpu-baseline --no-k7 \
  > gpurun_out/r01_launches.log 2>&1
grep -E "^  l" gpurun_out/r01_launches.log | head -3
for l in l3.b1.c2 l1.b0.c3 l1.b0.c2 l4.b1.c2; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 -o gpurun_out/r01_full_$l \
    python scripts/prof_layer.py --layer $l > gpurun_out/r01_full_$l.log 2>&1
  tail -1 gpurun_out/r01_full_$l.log
done

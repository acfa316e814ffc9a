# Round-1 profile evidence: timed bench (records tile picks), ncu launch list of
# the same bench command (kernel times + DRAM bytes per launch), and --set full
# captures of three representative layers with the bench's picks.
export CONV_Q_CACHE=$PWD/gpurun_out/tune_r50.json
rm -f $CONV_Q_CACHE
timeout 900 python bench.py --layers-out gpurun_out/layers_r50_int8.json > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err
cat gpurun_out/bench_r50.json | head -c 300; echo
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r01_launches.csv python bench.py --no-tune --steps 2 --warmup 3 --no-e2e --no-stem --no-cpu-baseline --no-k7 \
  > gpurun_out/r01_launches.log 2>&1
tail -2 gpurun_out/r01_launches.log; wc -l gpurun_out/r01_launches.csv
for l in l3.b1.c2 l1.b0.c3 l1.b0.c2 l4.b1.c2; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 -o gpurun_out/r01_full_$l \
    python scripts/prof_layer.py --layer $l > gpurun_out/r01_full_$l.log 2>&1
  tail -1 gpurun_out/r01_full_$l.log
done
timeout 300 ncu --set full --clock-control none -k regex:quantize -s 2 -c 1 -o gpurun_out/r01_full_quantize \
  python -c "
import torch, paper_2202_06819_b200 as cq
x = torch.randn(256, 56, 56, 64, device='cuda').half()
for _ in range(4): cq.quantize(x, 32.0, 8)
torch.cuda.synchronize()" > gpurun_out/r01_full_quantize.log 2>&1
ls -la gpurun_out/*.ncu-rep

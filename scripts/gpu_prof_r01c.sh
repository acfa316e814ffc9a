# Round-1 profile evidence (current build): timed bench (records tile picks), ncu launch
# list of the same bench command with those picks (kernel times + DRAM bytes per launch),
# --set full captures of representative layers, the stem and the quantize kernels.
export CONV_Q_CACHE=$PWD/gpurun_out/tune_r50.json
rm -f $CONV_Q_CACHE
timeout 900 python bench.py --layers-out gpurun_out/layers_r50_int8.json > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err
head -c 300 gpurun_out/bench_r50.json; echo
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r01_launches.csv python bench.py --no-tune --steps 2 --warmup 3 --no-e2e --no-stem --no-cpu-baseline --no-k7 \
  > gpurun_out/r01_launches.log 2>&1
wc -l gpurun_out/r01_launches.csv
for l in l3.b1.c2 l1.b0.c3 l1.b0.c2 l4.b1.c2 l3.b1.c3; do
  c=$(python -c "import json,sys; d=json.load(open('gpurun_out/layers_r50_int8.json'))['layers']; print([r['config'] for r in d if r['layer']=='$l'][0])")
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 -o gpurun_out/r01_full_$l \
    python scripts/prof_layer.py --layer $l --config $c > gpurun_out/r01_full_$l.log 2>&1
  tail -1 gpurun_out/r01_full_$l.log
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 -o gpurun_out/r01_full_stem \
    python scripts/prof_layer.py --layer stem > gpurun_out/r01_full_stem.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:quantize -s 2 -c 1 -o gpurun_out/r01_full_quantize \
  python -c "
import torch, paper_2202_06819_b200 as cq
x = torch.randn(256, 56, 56, 64, device='cuda').half()
for _ in range(4): cq.quantize(x, 32.0, 8)
torch.cuda.synchronize()" > gpurun_out/r01_full_quantize.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:s2d_quantize -s 2 -c 1 -o gpurun_out/r01_full_s2d_quantize \
  python -c "
import torch, paper_2202_06819_b200 as cq
p = cq.StemPlan(256, 224, 224, 3, 64, 7, 7, 3, 8)
x = torch.randn(256, 224, 224, 3, device='cuda').half()
for _ in range(4): p.quantize(x, 32.0)
torch.cuda.synchronize()" > gpurun_out/r01_full_s2d_quantize.log 2>&1
ls -la gpurun_out/*.ncu-rep
# summarise on the box (reports are too large to bring back), keep two reports
python scripts/launch_summary.py gpurun_out/r01_launches.csv resnet50_int8_b256 > gpurun_out/r01_launches_resnet50_int8_b256.txt 2>&1
for r in gpurun_out/r01_full_*.ncu-rep; do b=$(basename $r .ncu-rep); python scripts/ncu_summary.py $r > gpurun_out/$b.txt 2>&1; done
python scripts/ncu_src_top.py gpurun_out/r01_full_l3.b1.c3.ncu-rep $((256*14*14*1024)) > gpurun_out/r01_src_l3.b1.c3.txt 2>&1
python scripts/ncu_lines.py gpurun_out/r01_full_l3.b1.c3.ncu-rep 30 >> gpurun_out/r01_src_l3.b1.c3.txt 2>&1
python scripts/ncu_lines.py gpurun_out/r01_full_stem.ncu-rep 30 > gpurun_out/r01_src_stem.txt 2>&1
mkdir -p gpurun_out/keep; mv gpurun_out/r01_full_l3.b1.c2.ncu-rep gpurun_out/keep/ ; rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out

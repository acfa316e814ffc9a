#!/bin/bash
# Round-2 session-3 profile evidence (current build): the default bench line (as the driver runs it),
# the ncu launch list of the same command with the bench's tile picks, --set full summaries of
# representative layers, the stem and the max pool.  Summaries are written on the box.
O=gpurun_out/prof3; mkdir -p $O
export CONV_Q_CACHE=$PWD/$O/tune_r50.json
rm -f $CONV_Q_CACHE
timeout 900 python bench.py --layers-out $O/layers_r50.json > $O/bench_r50.json 2> $O/bench_r50.err
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv --log-file $O/launches.csv python bench.py --no-tune --no-graph --steps 2 --warmup 3 --no-e2e --no-parity --no-cpu-baseline --no-k7 \
  > $O/launches.log 2>&1
for l in l3.b1.c2 l3.b1.c3 l4.b1.c1 l1.b0.c3 l1.b0.c2; do
  c=$(python -c "import json,sys; d=json.load(open('$O/layers_r50.json'))['layers']; print([r['config'] for r in d if r['layer']=='$l'][0])")
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 -o $O/full_$l \
    python scripts/prof_layer.py --layer $l --config $c > $O/full_$l.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 -o $O/full_stem \
    python scripts/prof_layer.py --layer stem > $O/full_stem.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:maxpool -s 2 -c 1 -o $O/full_maxpool \
  python -c "
import torch, paper_2202_06819_b200 as cq
x = torch.randint(0, 255, (256, 112, 112, 64), dtype=torch.uint8, device='cuda')
for _ in range(4): cq.maxpool(x, 64, 3, 2, 1, 8)
torch.cuda.synchronize()" > $O/full_maxpool.log 2>&1
for r in $O/full_*.ncu-rep; do b=$(basename $r .ncu-rep); python scripts/ncu_summary.py $r > $O/r02s3_$b.txt 2>&1; done
python scripts/ncu_src_top.py $O/full_l3.b1.c3.ncu-rep $((256*14*14*1024)) > $O/r02s3_src_l3.b1.c3.txt 2>&1
rm -f $O/*.ncu-rep
python scripts/launch_summary.py $O/launches.csv resnet50_int8_b256 > $O/r02s3_launches.txt 2>&1; cp profiles/traffic_resnet50_int8_b256.json $O/ 2>/dev/null
for w in resnet50_int8_b256_res resnet50_int8_b256_uns resnet18_int4_b16 resnet18_int8_b1 resnet18_int4_b16_uns; do
  CONV_Q_CACHE=$O/cache_$w.json timeout 900 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --no-k7 --layers-out $O/layers_$w.json > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_r50_20.json 2> $O/bench_r50_20.err

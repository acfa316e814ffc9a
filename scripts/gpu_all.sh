# full GPU check: parity suite, default bench (as the driver runs it), INT4 and b1 workloads
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --layers-out gpurun_out/layers_r50_int8.json > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err
cat gpurun_out/bench_r50.json; grep -E "^  l|stem|e2e|step" gpurun_out/bench_r50.err | head -70
for w in resnet18_int4_b16 resnet18_int8_b1; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --no-k7 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  head -c 600 gpurun_out/bench_$w.json; echo
done

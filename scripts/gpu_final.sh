# parity suite, default bench (as the driver runs it), INT4 / batch-1 workloads, reference arm
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --layers-out gpurun_out/layers_r50_int8.json > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err; echo bench=$?
head -c 400 gpurun_out/bench_r50.json; echo
for w in resnet18_int4_b16 resnet18_int8_b1; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --no-k7 --layers-out gpurun_out/layers_$w.json > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  head -c 300 gpurun_out/bench_$w.json; echo
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; head -c 500 gpurun_out/bench_ref.json; echo
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"

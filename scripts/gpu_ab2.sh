# A/B on one box: current lib vs the previous commit's lib (bench step), alternating
for lib in libconvq.so libconvq_prev.so libconvq.so libconvq_prev.so; do
  CONV_Q_LIB=$PWD/paper_2202_06819_b200/$lib timeout 600 python bench.py --no-e2e --no-stem --no-cpu-baseline --no-k7 --steps 200 > gpurun_out/ab_$lib.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ab_$lib.json').read().strip().splitlines()[-1]); print('$lib', d['ms_per_step'], d['clocks']['sm_mhz'])"
done

# A/B: L2 policy of output stores (bench step, tuned once per setting)
for pol in 0 1 2 0; do
  CONV_Q_OUT_POLICY=$pol timeout 600 python bench.py --no-e2e --no-stem --no-cpu-baseline --no-k7 --steps 200 > gpurun_out/pol_$pol.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/pol_$pol.json').read().strip().splitlines()[-1]); print('policy $pol', d['value'], d['ms_per_step'])"
done

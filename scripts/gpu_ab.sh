# A/B the in-tree build against scratch/libconvq_old.so on the same box
for i in 1 2; do
  for lib in ${AB_LIBS:-scratch/libconvq_old.so paper_2202_06819_b200/libconvq.so}; do
    CONV_Q_LIB=$PWD/$lib timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-stem --no-k7 ${AB_ARGS} > gpurun_out/ab.json 2> gpurun_out/ab_$i_$(basename $lib).err
    echo "$lib $(python -c 'import json;d=json.load(open("gpurun_out/ab.json"));print(d["value"], d["ms_per_step"])')"
  done
done

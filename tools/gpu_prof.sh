#!/bin/bash
# One GPU call: FP64 peak microbenchmark + ncu --set full of the two kernels of the
# bench config(s).  Each ncu command line is first run plain (must exit 0).
mkdir -p gpurun_out
./tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1
for c in ${PCONFIGS:-c4 c5}; do
  case $c in c1|c3|c4) ks="kt_stage kt_grad";; *) ks="ks_stage ks_grad";; esac
  cmd="python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline"
  timeout 600 $cmd > gpurun_out/plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
  for k in $ks; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 \
      -o gpurun_out/prof_${c}_$k -f $cmd > gpurun_out/ncu_${c}_$k.log 2>&1
  done
done

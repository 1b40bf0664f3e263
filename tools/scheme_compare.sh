#!/bin/bash
# SDRT vs FR-SDRT vs FR-DG on the c4 workload (hex p=3 TGV), RK4 and the paper's RK54
mkdir -p gpurun_out
for sch in sdrt frsdrt frdg; do
  for it in rk4 rk54; do
    timeout 600 python bench.py --config c4 --scheme $sch --integrator $it --steps 20 --warmup 3 --no-cpu-baseline \
      > gpurun_out/cmp_${sch}_${it}.json 2> gpurun_out/cmp_${sch}_${it}.err
  done
done

#!/bin/bash
# SDRT vs FR-SDRT vs FR-DG on the simplex workloads (c5 tet p=3 TGV, c2 tri p=3 vortex)
mkdir -p gpurun_out
for c in c5 c2; do
  for sch in sdrt frsdrt frdg; do
    timeout 600 python bench.py --config $c --scheme $sch --steps 20 --warmup 3 --no-cpu-baseline \
      > gpurun_out/cmp_${c}_${sch}.json 2> gpurun_out/cmp_${c}_${sch}.err
  done
done

#!/bin/bash
# ncu --set full of one kernel (regex KREGEX) of one bench config, optionally under
# several environment settings (VARS="name:ENV=1 name2:ENV=0"); summaries are written on
# the box; only the report of the first setting is kept (size cap of gpurun_out).
mkdir -p gpurun_out
c=${CFG:-c4}; k=${KREGEX:-kt_grad}
cmd="python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline"
$cmd > gpurun_out/plain_$c.log 2>&1 || { echo "plain run failed"; exit 1; }
first=1
for ab in ${VARS:-default:X=1}; do
  name=${ab%%:*}; envs=${ab#*:}
  env ${envs//,/ } timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIP:-8} -c 1 \
    -o gpurun_out/prof_${c}_${name} -f $cmd > gpurun_out/ncu_${c}_$name.log 2>&1
  bash tools/ncu_summary.sh gpurun_out/prof_${c}_${name}.ncu-rep > gpurun_out/sum_${c}_${name}.txt 2>&1
  python tools/ncu_stalls.py gpurun_out/prof_${c}_${name}.ncu-rep > gpurun_out/stalls_${c}_${name}.txt 2>&1
  python tools/ncu_inst.py gpurun_out/prof_${c}_${name}.ncu-rep > gpurun_out/inst_${c}_${name}.txt 2>&1
  [ $first = 1 ] || rm -f gpurun_out/prof_${c}_${name}.ncu-rep
  first=0
done

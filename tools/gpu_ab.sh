#!/bin/bash
# One GPU call: GPU tests (optional subset via TESTSEL) then A/B bench lines of one config
# under a list of environment settings: AB="NAME1:ENV=1 NAME2:ENV=0" CFG=c4
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q ${TESTSEL:+-k "$TESTSEL"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
for c in ${CFG:-c4}; do
  for ab in ${AB:-default:X=1}; do
    name=${ab%%:*}; envs=${ab#*:}
    env ${envs//,/ } timeout 600 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline > gpurun_out/ab_${c}_$name.json 2> gpurun_out/ab_${c}_$name.err
  done
done

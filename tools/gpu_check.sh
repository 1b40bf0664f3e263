#!/bin/bash
# One GPU call: parity tests, bench lines for every config, ncu launch list of the bench.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-c4 c5 c3 c2 c1}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 ${BENCH_EXTRA} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
if [ -n "$NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
fi

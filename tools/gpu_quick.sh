#!/bin/bash
# One GPU call: parity tests (optionally a subset) + bench lines for selected configs.
mkdir -p gpurun_out
[ -x tools/fp64_peak ] && ./tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 900 python -m pytest tests -m gpu -x -q ${TESTSEL:+-k "$TESTSEL"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-c4 c5}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done

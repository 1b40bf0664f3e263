#!/bin/bash
# Round evidence in one GPU call: FP64 peak, full GPU tests, bench lines for every config
# (c4 = the default bench workload, with the CPU baseline), the ncu launch list of the
# default bench command, and ncu --set full captures of the two kernels of c4 and c5.
mkdir -p gpurun_out
./tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for c in c1 c2 c3 c5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
cmd="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline"
$cmd > gpurun_out/plain_launch.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv $cmd > gpurun_out/ncu_launch.log 2>&1
PCONFIGS="c4 c5" bash tools/gpu_prof.sh

#!/bin/bash
# Round-2 evidence in one GPU call: full GPU tests, smoke, bench lines for every config,
# compute-sanitizer (racecheck, memcheck) on small c1/c4/c5 runs, the ncu launch list of
# the default bench command and SASS/pipe counters of the dominant kernels.
O=gpurun_out/r2_ev; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in c1 c2 c3 c5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
cat > /tmp/san.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2105_08632_b200.solver import Solver
from sdrt_inputs import CONFIGS, initial_state
for name, N in (("c1", 4), ("c4", 3), ("c5", 3), ("c2", 4), ("c3", 3)):
    cfg = CONFIGS[name]
    S = Solver(cfg.etype, cfg.p, N, cfg.lo, cfg.hi, cfg.eq, **cfg.physics_kwargs())
    U = S.to_device(initial_state(cfg, S.sol_coords()))
    S.residual(U); S.rk_step(U, cfg.dt, 1)
    if name in ("c4", "c5"): S.rk54_step(U, cfg.dt, 1)
    torch.cuda.synchronize(); S.close()
print("sanitizer workload ok")
PY
for tool in racecheck memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san.py > $O/sanitizer_$tool.log 2>&1; echo "rc=$?" >> $O/sanitizer_$tool.log
done
cmd="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline"
$cmd > $O/plain_c4.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv $cmd > $O/ncu_launch.log 2>&1
M=gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed_op_dmma.sum,sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
for c in c4 c5 c3; do
  cmd="python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline"
  timeout 900 ncu --metrics $M --clock-control none -k regex:"k[ts]_" -s 6 -c 6 --csv --log-file $O/sass_$c.csv $cmd > $O/ncu_sass_$c.log 2>&1
done

#!/bin/bash
# Round-2 evidence (final code): GPU tests, smoke, bench lines for every config (+ the
# prism workload and the paper's RK54 protocol on c4), the ncu launch list of the default
# bench command, DMMA counters of c5.  PART=prof: ncu --set full captures of the two
# kernels of c4 and c5, summarised to text on the box (the .ncu-rep files are removed:
# gpurun returns at most 64 MiB).
O=gpurun_out/r2_fin; mkdir -p $O
if [ "$PART" = prof ]; then
  for c in c4 c5; do
    case $c in c4) ks="kt_grad kt_stage";; *) ks="ks_grad ks_stage";; esac
    cmd="python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline"
    for k in $ks; do
      rep=$O/prof_${c}_$k
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 -o $rep -f $cmd > $O/ncu_${c}_$k.log 2>&1
      { echo "ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 ($cmd), code at $(cat .commit 2>/dev/null)";
        bash tools/ncu_summary.sh $rep.ncu-rep; echo "-- stall reasons per source line"; python tools/ncu_stalls.py $rep.ncu-rep 12;
        echo "-- executed instructions"; python tools/ncu_inst.py $rep.ncu-rep 10; } > $O/r02_prof_${c}_${k}_summary.txt 2>&1
      rm -f $rep.ncu-rep
    done
  done
  exit 0
fi
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in c1 c2 c3 c5 c4pri; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --config c4 --integrator rk54 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c4_rk54.json 2> $O/bench_c4_rk54.err
for v in e4 e2; do
  SDRT_LIB=$PWD/paper_2105_08632_b200/libsdrt_$v.so timeout 600 python bench.py --config c2 --steps 50 --warmup 3 --no-cpu-baseline > $O/var_c2_$v.json 2> $O/var_c2_$v.err
done
SDRT_LIB=$PWD/paper_2105_08632_b200/libsdrt_e4.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_long.py -q -x -k c2 > $O/pytest_c2_e4.log 2>&1
cmd="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline"
$cmd > $O/plain_c4.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv $cmd > $O/ncu_launch.log 2>&1
M=gpu__time_duration.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"ks_" -s 6 -c 4 --csv --log-file $O/dmma_c5.csv python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_dmma.log 2>&1

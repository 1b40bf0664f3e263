#!/bin/bash
# Round-2 evidence at the current code (one GPU call): GPU tests, smoke, bench lines for
# every config (+ prisms, RK54 and the base two-sided-flux path on c4/c5 for comparison),
# the ncu launch list of the default bench command, SASS / DMMA / DRAM counters of the
# fused kernels (-> profiles/r02_sass_counts.json via tools/sass_counts.py) and ncu
# --set full summaries of the two kernels of c4 and c5 (reports removed: 64 MiB cap).
O=${O:-gpurun_out/r2c}; mkdir -p $O
git_commit=$(cat .commit 2>/dev/null)
if [ "$PART" != prof ]; then
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in c1 c2 c3 c5 c4pri; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --config c4 --integrator rk54 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c4_rk54.json 2> $O/bench_c4_rk54.err
for c in c4 c5; do
  SDRT_OSF=0 timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_${c}_twosided.json 2> $O/bench_${c}_twosided.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
cmd="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline"
$cmd > $O/plain_c4.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv $cmd > $O/ncu_launch.log 2>&1
M=gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
for c in c4 c5 c3; do
  cmd="python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline"
  timeout 900 ncu --metrics $M --clock-control none -k regex:"k[ts]_" -s 6 -c 6 --csv --log-file $O/sass_$c.csv $cmd > $O/ncu_sass_$c.log 2>&1
done
python tools/sass_counts.py $O/sass_counts.json c4=$O/sass_c4.csv c5=$O/sass_c5.csv c3=$O/sass_c3.csv > $O/sass_counts.log 2>&1
fi
if [ "$PART" != noprof ]; then
for c in c4 c5; do
  case $c in c4) ks="kt_grad kt_stage";; *) ks="ks_grad ks_stage";; esac
  cmd="python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline"
  for k in $ks; do
    rep=$O/prof_${c}_$k
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 9 -c 1 -o $rep -f $cmd > $O/ncu_${c}_$k.log 2>&1
    { echo "ncu --set full --clock-control none --import-source on -k regex:$k -s 9 -c 1 ($cmd), code at $git_commit";
      bash tools/ncu_summary.sh $rep.ncu-rep; echo "-- stall reasons per source line"; python tools/ncu_stalls.py $rep.ncu-rep 12;
      echo "-- executed instructions"; python tools/ncu_inst.py $rep.ncu-rep 10;
      echo "-- shared-memory wavefronts per source line"; python tools/ncu_smem.py $rep.ncu-rep 8; } > $O/r02_prof_${c}_${k}_summary.txt 2>&1
    rm -f $rep.ncu-rep
  done
done
fi

#!/bin/bash
# bench one config against each built tuning variant (libsdrt_<v>.so) and the default
mkdir -p gpurun_out
c=${1:-c5}; shift
for v in default "$@"; do
  if [ "$v" = default ]; then unset SDRT_LIB; else export SDRT_LIB=$PWD/paper_2105_08632_b200/libsdrt_$v.so; fi
  timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline > gpurun_out/var_${c}_$v.json 2> gpurun_out/var_${c}_$v.err
done

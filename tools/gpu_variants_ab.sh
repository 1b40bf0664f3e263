#!/bin/bash
# A/B of tuning-variant libraries (VS="v1 v2", libsdrt_<v>.so built with SDRT_VARIANT /
# SDRT_DEFS) against the default build on one config: GPU parity tests under the variants
# named in TESTV, then bench lines of default and variants, interleaved, REPS times.
O=gpurun_out/${OUT:-vab}; mkdir -p $O
lib() { echo /root/repo/paper_2105_08632_b200/libsdrt_$1.so; }
for v in $TESTV; do
  SDRT_LIB=$(lib $v) timeout 1200 python -m pytest tests -m gpu -x -q -k "${TESTSEL:-osf or parity or fused or guards}" > $O/pytest_$v.log 2>&1; echo "pytest rc=$?" >> $O/pytest_$v.log
done
for r in $(seq 1 ${REPS:-2}); do
  for c in ${CFG:-c4}; do
    timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/ab_${c}_default_$r.json 2> $O/ab_${c}_default_$r.err
    for v in $VS; do
      SDRT_LIB=$(lib $v) timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/ab_${c}_${v}_$r.json 2> $O/ab_${c}_${v}_$r.err
    done
  done
done

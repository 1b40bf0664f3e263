#!/bin/bash
# fused RK stage (SDRT_FUSE=1): parity tests, then c4 bench lines at several lags against
# the two-kernel stage
O=${O:-gpurun_out/fuse}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q > $O/pytest_fused.log 2>&1; echo "rc=$?" >> $O/pytest_fused.log
B="python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline"
timeout 300 $B > $O/bench_c4_base.json 2> $O/bench_c4_base.err
for lag in ${LAGS:-def 0 148 296 1184}; do
  if [ $lag = def ]; then SDRT_FUSE=1 timeout 300 $B > $O/bench_c4_fuse_$lag.json 2> $O/bench_c4_fuse_$lag.err
  else SDRT_FUSE=1 SDRT_FUSE_LAG=$lag timeout 300 $B > $O/bench_c4_fuse_$lag.json 2> $O/bench_c4_fuse_$lag.err; fi
done
for f in $O/bench_c4_*.json; do python - "$f" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    try: d = json.loads(l)
    except Exception: continue
    print(sys.argv[1], round(d["value"], 2), {k: round(v, 2) for k, v in d["kernel_ms"].items()})
PY
done

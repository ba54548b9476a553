#!/bin/bash
# Round-2 baseline capture of the round-1 final build: GPU tests, the default
# c5 line, and ncu --set full of the benched kernel AT c5 (k_step_co, a step
# launch, not the init) plus the traversal-ceiling kernel k_trace_bench.
TAG=${TAG:-r02a}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; tail -1 $OUT/pytest_gpu.log
fi
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err; cat $OUT/bench_c5.json | head -c 600; echo
cap() {   # name, kernel regex, launch-skip, command...
  local name=$1 re=$2 skip=$3; shift 3
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$re" --launch-skip $skip -c 1 \
      -o $OUT/$name "$@" > $OUT/ncu_$name.log 2>&1
  ncu -i $OUT/$name.ncu-rep --page raw --csv > $OUT/${name}_raw.csv 2>/dev/null
  ncu -i $OUT/$name.ncu-rep --page source --csv --print-source cuda,sass > $OUT/${name}_source.csv 2>/dev/null
  gzip -f $OUT/${name}_source.csv
  python tools/ncu_summary.py $OUT/${name}_raw.csv > $OUT/${name}_summary.txt 2>&1
  [ -n "$KEEP_REP" ] || rm -f $OUT/$name.ncu-rep
}
# c5: 8,388,608 chains, 2048^2; launch 0 is the INIT instantiation, 1.. are steps
cap k_step_co_c5 'k_step_co' 3 python tools/ncu_case.py clusters ra-quadtree lens 8388608 4 13 2048
cap k_trace_bench 'k_trace_bench' 1 python tools/trace_bench.py
du -sh $OUT
echo done

#!/bin/bash
# Wavefront step as the default: parity of the wf launch structure, the c5 line,
# launch list, ncu --set full of k_wf_trace and k_wf_logic at c5.
TAG=${TAG:-r02m}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_benched_path.py tests/test_gpu_parity.py -m gpu -x -q > $OUT/pytest_wf.log 2>&1; tail -3 $OUT/pytest_wf.log
timeout 900 python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.err; cat $OUT/bench_c5.json | cut -c1-1500
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file $OUT/launches_c5.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-relmse > $OUT/ncu_launch.log 2>&1
cap() {   # name, kernel regex, launch-skip, command...
  local name=$1 re=$2 skip=$3; shift 3
  timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$re" --launch-skip $skip -c 1 \
      -o $OUT/$name "$@" > $OUT/ncu_$name.log 2>&1
  ncu -i $OUT/$name.ncu-rep --page raw --csv > $OUT/${name}_raw.csv 2>/dev/null
  ncu -i $OUT/$name.ncu-rep --page source --csv --print-source cuda,sass > $OUT/${name}_source.csv 2>/dev/null
  gzip -f $OUT/${name}_source.csv
  python tools/ncu_summary.py $OUT/${name}_raw.csv > $OUT/${name}_summary.txt 2>&1
  python tools/ncu_lines.py $OUT/${name}_source.csv.gz 30 > $OUT/${name}_lines.txt 2>&1
  [ -n "$KEEP_REP" ] || rm -f $OUT/$name.ncu-rep
}
cap k_wf_trace_c5 'k_wf_trace' 1 python tools/ncu_case.py clusters ra-quadtree lens 8388608 2 13 2048
cap k_wf_logic_c5 'k_wf_logic' 2 python tools/ncu_case.py clusters ra-quadtree lens 8388608 2 13 2048
cat $OUT/k_wf_trace_c5_summary.txt $OUT/k_wf_logic_c5_summary.txt
du -sh $OUT
echo done

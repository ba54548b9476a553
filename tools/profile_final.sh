#!/bin/bash
# End-of-round capture: GPU tests, every bench line (with CPU baselines), the
# reference arm, the default command's launch list, and one ncu --set full of
# each workload's dominant kernel (exported to CSV on the box; the .ncu-rep
# files are dropped unless KEEP_REP=1 so the output stays under gpurun's cap).
TAG=${TAG:-r01n}
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ -z "$SKIP_TESTS" ]; then
  python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -1 $OUT/pytest_gpu.log
  python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
fi
python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.err
python bench.py --impl reference > $OUT/bench_ref_c5.json 2> $OUT/bench_ref_c5.err
for w in c4 c3 c2 c1; do python bench.py --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.err; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches_c5.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
cap() {   # name, kernel regex, launch-skip, command...
  local name=$1 re=$2 skip=$3; shift 3
  ncu --set full --clock-control none --import-source on -k "regex:$re" --launch-skip $skip -c 1 \
      -o $OUT/$name "$@" > $OUT/ncu_$name.log 2>&1
  ncu -i $OUT/$name.ncu-rep --page raw --csv > $OUT/${name}_raw.csv 2>/dev/null
  ncu -i $OUT/$name.ncu-rep --page source --csv --print-source cuda,sass > $OUT/${name}_source.csv 2>/dev/null
  gzip -f $OUT/${name}_source.csv
  [ -n "$KEEP_REP" ] || rm -f $OUT/$name.ncu-rep
}
cap k_step_co_c4 k_step_co 1 python tools/ncu_case.py clusters ra-quadtree lens 1048576 2 13 1024
cap k_mix_coop_c2 k_mix_coop 1 python bench.py --workload c2 --steps 1024 --no-cpu-baseline
cap k_step_c3 '^k_step$' 0 python tools/ncu_case.py caustic ra-quadtree multi-chain 262144 2 17 512
for f in $OUT/bench_*.json; do python -c "import json,sys;d=json.load(open(sys.argv[1]));r=d.get('roofline') or {};print(sys.argv[1],d['value'],d.get('e2e',{}).get('value'),r.get('frac'),r.get('kernel_share'))" $f; done
du -sh $OUT
echo done

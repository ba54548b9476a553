#!/bin/bash
# Full capture of the wavefront build: GPU tests, smoke, every bench line, reference arm,
# launch list of the default command, ncu --set full of k_wf_trace / k_wf_logic at c5
# (a mid-step round: launch-skip past the full first rounds), c3 / c2 kernels, 2-rank gloo run.
TAG=${TAG:-r02y}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
timeout 900 python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.err; cut -c1-300 $OUT/bench_c5.json
if [ -z "$SKIP_TESTS" ]; then
  timeout 2700 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -1 $OUT/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
fi
timeout 900 python bench.py --impl reference > $OUT/bench_ref_c5.json 2> $OUT/bench_ref_c5.err
for w in c4 c3 c2 c1; do timeout 900 python bench.py --workload $w --no-relmse > $OUT/bench_$w.json 2> $OUT/bench_$w.err; done
RAMLT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus 2 --workload c4 --steps 8 > $OUT/bench_c4_gloo2.json 2> $OUT/bench_c4_gloo2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file $OUT/launches_c5.csv \
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
cap k_wf_trace_c5_bounce 'k_wf_trace' 5 python tools/ncu_case.py clusters ra-quadtree lens 8388608 2 13 2048
cap k_wf_logic_c5 'k_wf_logic' 2 python tools/ncu_case.py clusters ra-quadtree lens 8388608 2 13 2048
cap k_wf_logic_c5_bounce 'k_wf_logic' 5 python tools/ncu_case.py clusters ra-quadtree lens 8388608 2 13 2048
cap k_wf_bounce_c5 'k_wf_bounce' 4 python tools/ncu_case.py clusters ra-quadtree lens 8388608 2 13 2048
for f in $OUT/bench_*.json; do python -c "import json,sys;d=json.load(open(sys.argv[1]));r=d.get('roofline') or {};print(sys.argv[1],d.get('value'),(d.get('e2e') or {}).get('value'),r.get('frac'),r.get('kernel_share'))" $f; done
timeout 600 python tools/e2e_phases.py c5 128 2>&1 | tail -1 | tee $OUT/e2e_phases_c5.txt
RAMLT_WF_LOG=1 timeout 600 python tools/ncu_case.py clusters ra-quadtree lens 8388608 2 13 2048 > $OUT/wf_log_c5.txt 2>&1
du -sh $OUT
echo done
echo done2

#!/bin/bash
# End-of-round capture: GPU tests, every bench line (with CPU baselines), the
# reference arm, the default command's launch list, and one ncu --set full of
# each workload's dominant kernel.  Output: gpurun_out/$TAG/.
TAG=${TAG:-r01n}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -1 $OUT/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.err
python bench.py --impl reference > $OUT/bench_ref_c5.json 2> $OUT/bench_ref_c5.err
for w in c4 c3 c2 c1; do python bench.py --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.err; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches_c5.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_step_co --launch-skip 1 -c 1 \
    -o $OUT/k_step_co_c4 python tools/ncu_case.py clusters ra-quadtree lens 1048576 2 13 1024 > $OUT/ncu_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_mix_coop --launch-skip 1 -c 1 \
    -o $OUT/k_mix_coop_c2 python bench.py --workload c2 --steps 1024 --no-cpu-baseline > $OUT/ncu_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'^k_step$' -c 1 -o $OUT/k_step_c3 \
    python tools/ncu_case.py caustic ra-quadtree multi-chain 262144 2 17 512 > $OUT/ncu_c3.log 2>&1
for f in $OUT/bench_*.json; do python -c "import json,sys;d=json.load(open(sys.argv[1]));r=d.get('roofline') or {};print(sys.argv[1],d['value'],d.get('e2e',{}).get('value'),r.get('frac'),r.get('kernel_share'))" $f; done
echo done

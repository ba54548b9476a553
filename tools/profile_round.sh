#!/bin/bash
# Round profile: bench lines (c5 default, c4, c3, c2), the launch list of the
# default bench command, and one `ncu --set full` capture of each workload's
# top kernel.  Output: gpurun_out/$TAG/ (copy what is judged into profiles/).
# SKIP_BENCH=1 skips the bench lines; NCU=0 skips the captures.
TAG=${TAG:-r01e}
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ -z "$SKIP_BENCH" ]; then
  python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.err || exit 1
  python bench.py --workload c4 > $OUT/bench_c4.json 2> $OUT/bench_c4.err || exit 1
  python bench.py --workload c3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err || exit 1
  python bench.py --workload c2 > $OUT/bench_c2.json 2> $OUT/bench_c2.err || exit 1
fi
[ "$NCU" = "0" ] && { echo done; exit 0; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c5.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
python tools/ncu_case.py clusters ra-quadtree lens 1048576 2 13 1024 || exit 1
# the step kernel (launch 0 of k_step_co is chain initialisation)
ncu --set full --clock-control none --import-source on -k regex:k_step_co --launch-skip 1 -c 1 \
    -o $OUT/k_step_co_c4 python tools/ncu_case.py clusters ra-quadtree lens 1048576 2 13 1024 > $OUT/ncu_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_mix_coop -c 1 \
    -o $OUT/k_mix_coop_c2 python bench.py --workload c2 --steps 1024 --no-cpu-baseline > $OUT/ncu_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'^k_step$' -c 1 -o $OUT/k_step_c3 \
    python tools/ncu_case.py caustic ra-quadtree multi-chain 262144 2 17 512 > $OUT/ncu_c3.log 2>&1
echo done

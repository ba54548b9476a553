#!/bin/bash
# 32 B state chunks / smem-resident state / planned rounds: A/B + launch list of the new wavefront
OUT=gpurun_out/r02o; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_benched_path.py -m gpu -x -q -k "bvh_equals or reference_c1" > $OUT/pytest_wf.log 2>&1; tail -2 $OUT/pytest_wf.log
timeout 1500 python tools/ab.py c5 "" c16 smem "@RAMLT_WF_POLL=1" 2>&1 | tail -5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file $OUT/launches.csv \
    python tools/ncu_case.py clusters ra-quadtree lens 8388608 4 13 2048 > $OUT/ncu_launch.log 2>&1
tail -2 $OUT/ncu_launch.log

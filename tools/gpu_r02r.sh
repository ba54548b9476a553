#!/bin/bash
# Brute-force wavefront (c3), rebuilt BVH builder / parser parity, e2e phase breakdown, ray-order probe.
OUT=gpurun_out/r02r; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wf" > $OUT/pytest_wf.log 2>&1; tail -2 $OUT/pytest_wf.log
timeout 900 python -m pytest tests/test_gpu_benched_path.py -m gpu -x -q > $OUT/pytest_benched.log 2>&1; tail -2 $OUT/pytest_benched.log
timeout 900 python tools/ab.py c3 "" "@RAMLT_STEP_KERNEL=wf" 2>&1 | tail -3 | tee $OUT/ab_c3.txt
timeout 600 python tools/e2e_phases.py c5 128 2>&1 | tail -1 | tee $OUT/e2e_phases_c5.txt
timeout 600 python tools/e2e_phases.py c3 256 2>&1 | tail -1 | tee $OUT/e2e_phases_c3.txt
for c in 0 8 32; do RAMLT_TB_CELLS=$c timeout 300 python tools/trace_bench.py 2>&1 | tail -1 | sed "s/^/cells=$c /"; done | tee $OUT/ray_order.txt

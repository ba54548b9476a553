#!/bin/bash
# batched visibility yields in the wavefront step: parity first, then A/B against the fused coroutine kernel
OUT=gpurun_out/r02n; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_benched_path.py tests/test_gpu_parity.py -m gpu -x -q -k "wf or wavefront or bvh or benched or full_scene or reference_c1 or matches_f64 or acceptance" > $OUT/pytest_wf.log 2>&1; tail -5 $OUT/pytest_wf.log
timeout 1500 python tools/ab.py c5 "" "@RAMLT_STEP_KERNEL=co" "@M_REFINE=10000000" "@RAMLT_WF_REFILL=4" "@RAMLT_WF_REFILL=16" 2>&1 | tail -12

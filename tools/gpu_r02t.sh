#!/bin/bash
# Wavefront chain initialisation: parity, init time (e2e phases) against the fused kernel, per-round queue lengths.
OUT=gpurun_out/r02t; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wf" > $OUT/pytest_wf.log 2>&1; tail -2 $OUT/pytest_wf.log
timeout 1200 python -m pytest tests/test_gpu_benched_path.py -m gpu -x -q > $OUT/pytest_benched.log 2>&1; tail -2 $OUT/pytest_benched.log
timeout 600 python tools/e2e_phases.py c5 32 2>&1 | tail -1 | tee $OUT/e2e_phases_c5_wfinit.txt
RAMLT_INIT_KERNEL=co timeout 600 python tools/e2e_phases.py c5 32 2>&1 | tail -1 | tee $OUT/e2e_phases_c5_coinit.txt
timeout 600 python tools/e2e_phases.py c4 32 2>&1 | tail -1 | tee $OUT/e2e_phases_c4_wfinit.txt
RAMLT_INIT_KERNEL=co timeout 600 python tools/e2e_phases.py c4 32 2>&1 | tail -1 | tee $OUT/e2e_phases_c4_coinit.txt
RAMLT_WF_LOG=1 RAMLT_INIT_KERNEL=co timeout 600 python tools/ncu_case.py clusters ra-quadtree lens 8388608 2 13 2048 > $OUT/wf_log_c5.txt 2>&1; head -20 $OUT/wf_log_c5.txt
RAMLT_WF_LOG=1 timeout 600 python tools/ncu_case.py clusters ra-quadtree lens 1048576 1 13 1024 2>&1 | grep "wf init" | awk 'NR<=12 || NR%50==0' | tee $OUT/wf_log_init_c4.txt | tail -15

#!/bin/bash
# Compact bounce image (all precisions / RNGs) + the bounce loop as its own kernel (RAMLT_WF_BOUNCE=1):
# parity of both, A/B against the 4-hot-sector build (hc2).
OUT=gpurun_out/r02x; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wf" > $OUT/pytest_wf.log 2>&1; tail -2 $OUT/pytest_wf.log
RAMLT_WF_BOUNCE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wf" > $OUT/pytest_wf_bounce.log 2>&1; tail -2 $OUT/pytest_wf_bounce.log
timeout 1500 python -m pytest tests/test_gpu_benched_path.py -m gpu -x -q -k "not slow" > $OUT/pytest_benched.log 2>&1; tail -2 $OUT/pytest_benched.log
RAMLT_WF_BOUNCE=1 timeout 1500 python -m pytest tests/test_gpu_benched_path.py -m gpu -x -q -k "not slow" > $OUT/pytest_benched_bounce.log 2>&1; tail -2 $OUT/pytest_benched_bounce.log
timeout 1500 python tools/ab.py c5 "" hc2 "@RAMLT_WF_BOUNCE=1" 2>&1 | tail -4 | tee $OUT/ab_c5.txt
timeout 900 python tools/ab.py c4 "" hc2 "@RAMLT_WF_BOUNCE=1" 2>&1 | tail -4 | tee $OUT/ab_c4.txt

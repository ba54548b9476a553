#!/bin/bash
# Per-yield-point chain queues: parity of the wavefront launch structure + A/B against the single queue (base).
OUT=gpurun_out/r02s; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wf" > $OUT/pytest_wf.log 2>&1; tail -2 $OUT/pytest_wf.log
timeout 1200 python -m pytest tests/test_gpu_benched_path.py tests/test_gpu_multi.py -m gpu -x -q > $OUT/pytest_benched.log 2>&1; tail -2 $OUT/pytest_benched.log
timeout 1500 python tools/ab.py c5 "" base 2>&1 | tail -3 | tee $OUT/ab_c5.txt
timeout 900 python tools/ab.py c4 "" base 2>&1 | tail -3 | tee $OUT/ab_c4.txt

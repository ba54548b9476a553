#!/bin/bash
# Hot/cold coroutine state (bounce-loop chains move 4 of 10 sectors): parity + A/B against the full-state build (mq2).
OUT=gpurun_out/r02v; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wf or co" > $OUT/pytest_wf.log 2>&1; tail -2 $OUT/pytest_wf.log
timeout 1500 python -m pytest tests/test_gpu_benched_path.py tests/test_gpu_multi.py -m gpu -x -q > $OUT/pytest_benched.log 2>&1; tail -2 $OUT/pytest_benched.log
timeout 1500 python tools/ab.py c5 "" mq2 2>&1 | tail -3 | tee $OUT/ab_c5.txt
timeout 900 python tools/ab.py c4 "" mq2 2>&1 | tail -3 | tee $OUT/ab_c4.txt

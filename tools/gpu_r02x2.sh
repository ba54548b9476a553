#!/bin/bash
OUT=gpurun_out/r02x2; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_benched_path.py -m gpu -q -k "not slow" > $OUT/pytest_benched.log 2>&1; tail -3 $OUT/pytest_benched.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py -m gpu -x -q > $OUT/pytest_parity_multi.log 2>&1; tail -3 $OUT/pytest_parity_multi.log

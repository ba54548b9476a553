#!/bin/bash
# New round-2 GPU tests + the default bench line (quick iteration script).
TAG=${TAG:-r02b}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1500 python -m pytest ${TESTS:-tests/test_gpu_multi.py tests/test_gpu_benched_path.py} -q -s -rA \
    > $OUT/pytest_new.log 2>&1; tail -30 $OUT/pytest_new.log
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.err; head -c 3000 $OUT/bench_c5.json; tail -3 $OUT/bench_c5.err
fi
echo done

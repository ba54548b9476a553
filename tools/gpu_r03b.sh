#!/bin/bash
# Re-verification of the final tree (r02y build + the INIT instantiations of the compact image / k_wf_bounce).
OUT=gpurun_out/r03b; mkdir -p $OUT
timeout 2700 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -1 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.err; cut -c1-200 $OUT/bench_c5.json
timeout 900 python bench.py --impl reference > $OUT/bench_ref_c5.json 2> $OUT/bench_ref_c5.err; cut -c1-200 $OUT/bench_ref_c5.json

#!/bin/bash
# Chain initialisation as wavefront rounds with the compact image + k_wf_bounce<INIT>: parity, init time vs the fused kernel.
OUT=gpurun_out/r02z; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wf" > $OUT/pytest_wf.log 2>&1; tail -2 $OUT/pytest_wf.log
timeout 900 python -m pytest tests/test_gpu_benched_path.py -m gpu -x -q -k "not slow" > $OUT/pytest_benched.log 2>&1; tail -2 $OUT/pytest_benched.log
RAMLT_INIT_KERNEL=wf timeout 600 python tools/e2e_phases.py c5 16 2>&1 | tail -1 | tee $OUT/e2e_phases_c5_wfinit.txt
RAMLT_INIT_KERNEL=co timeout 600 python tools/e2e_phases.py c5 16 2>&1 | tail -1 | tee $OUT/e2e_phases_c5_coinit.txt
RAMLT_INIT_KERNEL=wf timeout 600 python tools/e2e_phases.py c4 16 2>&1 | tail -1 | tee $OUT/e2e_phases_c4_wfinit.txt
RAMLT_INIT_KERNEL=co timeout 600 python tools/e2e_phases.py c4 16 2>&1 | tail -1 | tee $OUT/e2e_phases_c4_coinit.txt

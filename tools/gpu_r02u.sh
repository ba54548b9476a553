#!/bin/bash
# Two concurrent wavefront pipelines: parity against the single pipeline, A/B at c5 with block-budget variants.
OUT=gpurun_out/r02u; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_benched_path.py -m gpu -x -q -k "pipelines" > $OUT/pytest_pipes.log 2>&1; tail -3 $OUT/pytest_pipes.log
timeout 2400 python tools/ab.py c5 "" "@RAMLT_WF_PIPES=2" "@RAMLT_WF_PIPES=2,RAMLT_WF_LBLK=3,RAMLT_WF_TBLK=4" "@RAMLT_WF_PIPES=2,RAMLT_WF_LBLK=2,RAMLT_WF_TBLK=5" "@RAMLT_WF_PIPES=2,RAMLT_WF_LBLK=3,RAMLT_WF_TBLK=6" 2>&1 | tail -5 | tee $OUT/ab_c5_pipes.txt

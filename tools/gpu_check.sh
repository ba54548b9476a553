#!/bin/bash
# GPU parity suite + c4 probes (default kernel choice) -- quick check after a
# kernel change.  VARIANTS="x y" also probes paper_2402_08273_b200/_lib/libramlt_gpu_<v>.so.
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
timeout 300 python tools/probe.py c4 2>&1 | grep "mut/s" | sed "s/^/default: /"
for v in $VARIANTS; do
  RAMLT_GPU_LIB=$PWD/paper_2402_08273_b200/_lib/libramlt_gpu_$v.so timeout 300 python tools/probe.py c4 2>&1 | grep "mut/s" | sed "s/^/$v: /"
done
timeout 300 python tools/e2e_phases.py c4

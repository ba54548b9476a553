#!/bin/bash
# Sweep the coroutine kernel's BVH knobs on c4 (tools/probe.py c4).
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "co" 2>&1 | tail -2
for pv in smem global; do for r in 4 8 16 24; do
  RAMLT_STEP_KERNEL=co RAMLT_CO_PV=$pv RAMLT_CO_REFILL=$r timeout 300 python tools/probe.py c4 2>&1 | grep "mut/s" | sed "s/^/co pv=$pv refill=$r: /"
done; done

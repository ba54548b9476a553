#!/bin/bash
# potential of ray sorting: k_trace_bench on the same ray population in (cell, octant) bucket order
for c in 0 4 8 16 32; do RAMLT_TB_CELLS=$c timeout 300 python tools/trace_bench.py 2>&1 | tail -1 | sed "s/^/cells=$c /"; done

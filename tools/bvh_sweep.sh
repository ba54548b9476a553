#!/bin/bash
# BVH build-quality sweep on the c4 scene: traversal probe + c4 step throughput
# per builder setting (RAMLT_BVH_BINS / RAMLT_BVH_CT / RAMLT_BVH_LEAF).
for cfg in "16 0 4" "32 0 4" "32 1 2" "32 2 2" "32 1 4" "16 0 8" "32 0.5 2"; do
  set -- $cfg
  export RAMLT_BVH_BINS=$1 RAMLT_BVH_CT=$2 RAMLT_BVH_LEAF=$3
  t=$(python tools/trace_bench.py 2>&1 | grep rays/s | sed 's/refill=8: //')
  p=$(timeout 300 python -c "
import sys; sys.argv=['x']; sys.path.insert(0,'tools'); import probe; probe.probe_c4()" 2>&1 | grep -o "[0-9.]* M mut/s")
  echo "bins=$1 ct=$2 leaf=$3: trace $t | c4 $p"
done

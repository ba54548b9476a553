#!/bin/bash
# BVH leaf size on the final wavefront build (trace = 72 % of the step).
OUT=gpurun_out/r03a; mkdir -p $OUT
timeout 1500 python tools/ab.py c5 "" "@RAMLT_BVH_LEAF=2" "@RAMLT_BVH_LEAF=3" "@RAMLT_BVH_LEAF=6" 2>&1 | tail -4 | tee $OUT/ab_c5_leaf.txt

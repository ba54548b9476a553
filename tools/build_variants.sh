#!/bin/bash
# Build A/B variants of libramlt_gpu.so: tools/build_variants.sh name "NVEXTRA flags" [name "flags" ...]
# -> paper_2402_08273_b200/_lib/libramlt_gpu_<name>.so (RAMLT_GPU_LIB selects one).
cd "$(dirname "$0")/../paper_2402_08273_b200/csrc"
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  ( make -s -j4 OUT=/tmp/ramlt_var_$name NVEXTRA="$flags" > /tmp/ramlt_var_$name.log 2>&1 &&
    cp /tmp/ramlt_var_$name/libramlt_gpu.so ../_lib/libramlt_gpu_$name.so && echo "built $name" ) &
done
wait

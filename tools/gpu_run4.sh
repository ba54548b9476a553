python tools/ncu_case.py caustic ra-quadtree multi-chain 262144 6 > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/prof_co python tools/ncu_case.py caustic ra-quadtree multi-chain 262144 6 > gpurun_out/ncu4.log 2>&1; echo ncu=$?
RAMLT_STEP_KERNEL=mega ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/prof_mega python tools/ncu_case.py caustic ra-quadtree multi-chain 262144 6 > gpurun_out/ncu4m.log 2>&1; echo ncu=$?

#!/bin/bash
# Key warp-efficiency metrics of the c4 step kernels (mega vs coroutine).
M=smsp__thread_inst_executed_per_inst_executed.ratio,smsp__inst_executed.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct
python tools/ncu_case.py clusters ra-quadtree lens 1048576 2 13 1024 || exit 1
ncu --metrics $M --clock-control none -k regex:k_step -c 2 --csv python tools/ncu_case.py clusters fixed lens 1048576 2 13 1024 > gpurun_out/ncu_mega.csv 2>&1
RAMLT_STEP_KERNEL=co RAMLT_CO_PV=global RAMLT_CO_REFILL=4 ncu --metrics $M --clock-control none -k regex:k_step -c 2 --csv python tools/ncu_case.py clusters fixed lens 1048576 2 13 1024 > gpurun_out/ncu_co4.csv 2>&1
RAMLT_STEP_KERNEL=co RAMLT_CO_PV=global RAMLT_CO_REFILL=32 ncu --metrics $M --clock-control none -k regex:k_step -c 2 --csv python tools/ncu_case.py clusters fixed lens 1048576 2 13 1024 > gpurun_out/ncu_co32.csv 2>&1

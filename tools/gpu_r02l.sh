# wavefront step (k_wf_logic / k_wf_trace) vs the coroutine kernel; plain 64 B nodes + 64 B triangles, new builder
timeout 1200 python -m pytest tests/test_gpu_benched_path.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r02l_pytest.log 2>&1; tail -3 gpurun_out/r02l_pytest.log
timeout 300 python tools/trace_bench.py 2>&1 | tail -1
timeout 2000 python tools/ab.py c5 "" "@RAMLT_STEP_KERNEL=co" wf10 wf8 "@RAMLT_WF_REFILL=4" "@RAMLT_WF_REFILL=16" 2>&1 | tail -20

python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python tools/probe.py > gpurun_out/probe.log 2>&1; echo probe=$?; cat gpurun_out/probe.log
RAMLT_STEP_KERNEL=mega timeout 300 python tools/probe.py > gpurun_out/probe_mega.log 2>&1; echo probe_mega=$?; cat gpurun_out/probe_mega.log

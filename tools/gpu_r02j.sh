set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02j_pytest.log 2>&1; tail -3 gpurun_out/r02j_pytest.log
timeout 600 python bench.py > gpurun_out/r02j_bench_c5.json 2> gpurun_out/r02j_bench_c5.err; cat gpurun_out/r02j_bench_c5.json
timeout 300 python tools/trace_bench.py > gpurun_out/r02j_trace.txt 2>&1; cat gpurun_out/r02j_trace.txt

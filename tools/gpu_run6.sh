python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke=$?; cat gpurun_out/smoke.log
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench=$?; cat gpurun_out/bench_c3.json; tail -2 gpurun_out/bench_c3.err
python bench.py --workload c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench_c1=$?; cat gpurun_out/bench_c1.json
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c3.json 2>&1; cat gpurun_out/bench_ref_c3.json
python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k_step -s 6 -c 1 -o gpurun_out/prof_c3 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?

timeout 900 python tools/ab.py c3 scan1 "" 2>&1 | grep "mean\|rror"
for v in "" scan1; do
  lib=""; [ -n "$v" ] && lib="RAMLT_GPU_LIB=$PWD/paper_2402_08273_b200/_lib/libramlt_gpu_$v.so"
  env $lib timeout 300 python bench.py --workload c1 --no-cpu-baseline --no-relmse 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 $v', round(d['value']/1e6,2), 'M/s frac', round(d['roofline']['frac'],4))"
done
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_statistics.py tests/test_gpu_benched_path.py -k "not full_scene and not at_scale and not unmodified" 2>&1 | tail -2

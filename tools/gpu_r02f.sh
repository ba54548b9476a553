timeout 900 python tools/ab.py c3 base "" 2>&1 | grep "mean\|rror"
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_benched_path.py -k "not full_scene and not at_scale and not unmodified" 2>&1 | tail -2

for v in mega co co_static; do echo "== $v"; RAMLT_STEP_KERNEL=$v timeout 300 python tools/probe.py 2>&1 | grep -E "262144|G= 1"; done
python -m pytest tests/test_gpu_parity.py -q --timeout 300 -p no:cacheprovider -x 2>&1 | tail -2

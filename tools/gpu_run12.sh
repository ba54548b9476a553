python -m pytest tests/test_gpu_parity.py -q --timeout 600 -p no:cacheprovider -k "bvh" 2>&1 | tail -2
for L in 2 4 8; do RAMLT_BVH_LEAF=$L timeout 600 python tools/probe.py c4 2>&1 | tail -2 | sed "s/^/leaf$L: /"; done

# BVH layout A/B: base (round-2 layout), default (quantised 32 B nodes + 64 B triangles, 64 SAH bins, large
# triangles isolated at the root), default@old-builder, p (64 B nodes + 64 B triangles, old builder)
L=$PWD/paper_2402_08273_b200/_lib
timeout 1200 python -m pytest tests/test_gpu_benched_path.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r02k_pytest.log 2>&1; tail -3 gpurun_out/r02k_pytest.log
for v in base default oldbuild p; do
  unset RAMLT_GPU_LIB RAMLT_BVH_BINS RAMLT_BVH_ISOLATE
  case $v in base|p) export RAMLT_GPU_LIB=$L/libramlt_gpu_$v.so;; oldbuild) export RAMLT_BVH_BINS=32 RAMLT_BVH_ISOLATE=0;; esac
  echo "== $v"; timeout 300 python tools/trace_bench.py 2>&1 | tail -1
done
unset RAMLT_GPU_LIB RAMLT_BVH_BINS RAMLT_BVH_ISOLATE
timeout 1500 python tools/ab.py c5 base "" p "@RAMLT_BVH_BINS=32,RAMLT_BVH_ISOLATE=0" 2>&1 | tail -12

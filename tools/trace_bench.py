"""Traversal-only throughput of the BVH on the c4/c5 scene (ramlt_gpu_trace_benchmark):
incoherent closest-hit rays per second, the ceiling a ray-tracing kernel of this
design can reach, next to the chain-step kernel's effective rays/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_08273_b200 import Engine, RenderConfig, scenes  # noqa: E402

text = scenes.cluster_room(n_tris=1 << 20)
for refill in (os.environ.get("REFILLS") or "8").split():
    os.environ["RAMLT_CO_REFILL"] = refill
    eng = Engine(text, RenderConfig(strategy="fixed", chains=1024, mutations=1024, width=64, height=64,
                                    max_vertices=13, precision="f32", rng="philox"))
    eng.trace_benchmark(1 << 22)
    n = 1 << 26
    ms, hits = eng.trace_benchmark(n)
    print(f"refill={refill}: {n / (ms / 1e3) / 1e6:.1f} M rays/s ({ms:.1f} ms for {n} rays, hit {hits / n:.3f})",
          flush=True)
    eng.close()

import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2402_08273_b200 import Engine, RenderConfig, scenes
for prec, rng in (("f32", "philox"), ("f64", "philox"), ("f64", "pcg32")):
    for target in (0.5,):
        cfg = RenderConfig(strategy="global", perturbation="lens", chains=1000, mutations=3_000_000,
                           width=64, height=64, max_vertices=9, b_samples=100000, seed=5,
                           target_acceptance=target, metrics_interval=300_000, trace_enabled=True,
                           trace_capacity=1 << 21, precision=prec, rng=rng)
        eng = Engine(scenes.cornell_box(), cfg)
        eng.estimate_b(); eng.init_chains(); eng.run(cfg.mutations)
        m = eng.metrics(); tr = eng.trace(); lam, n = eng.regions()
        print(prec, rng, "acc per interval", np.round(m[:, 3], 3), "lambda", lam[0], "n", n[0],
              "trace lambdas", np.round(tr[:12, 3], 2), tr.shape)
        eng.close()

import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2402_08273_b200 import Engine, RenderConfig, scenes
def run(prec, rng, strategy="global", lam=1.0, chains=1000, muts=1_500_000, lanes=0, env=None):
    if env:
        os.environ.update(env)
    cfg = RenderConfig(strategy=strategy, perturbation="lens", chains=chains, mutations=muts,
                       width=64, height=64, max_vertices=9, b_samples=100000, seed=5, lambda_init=lam,
                       target_acceptance=0.5, metrics_interval=muts // 5, precision=prec, rng=rng, lanes_per_chain=lanes)
    eng = Engine(scenes.cornell_box(), cfg)
    eng.estimate_b(); eng.init_chains(); eng.run(cfg.mutations)
    m = eng.metrics(); lam_, n = eng.regions()
    eng.close()
    if env:
        for k in env: os.environ.pop(k)
    return np.round(m[:, 3], 3), lam_[0]
print("f32 pcg global", run("f32", "pcg32"))
print("f32 philox global nocoop", run("f32", "philox", env={"RAMLT_COOP": "0"}))
print("f32 philox global G=1", run("f32", "philox", lanes=1))
for lam in (-4.0, -5.5, -8.0, -15.0, -30.0):
    print("f32 philox fixed", lam, run("f32", "philox", strategy="fixed", lam=lam, muts=200_000))
    print("f64 philox fixed", lam, run("f64", "philox", strategy="fixed", lam=lam, muts=200_000))

import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2402_08273_b200 import Engine, RenderConfig, scenes
res = {}
for prec in ("f64", "f32"):
    cfg = RenderConfig(strategy="fixed", perturbation="lens", chains=2000, mutations=2000 * 4, width=64, height=64,
                       max_vertices=9, b_samples=10000, seed=5, lambda_init=-5.0, precision=prec, rng="pcg32",
                       log_steps=4, lanes_per_chain=1)
    eng = Engine(scenes.cornell_box(), cfg)
    eng.set_b(1.0); eng.init_chains(); eng.run(cfg.mutations)
    a, f = eng.decisions(4)
    res[prec] = (a, f)
    eng.close()
a64, f64 = res["f64"]; a32, f32 = res["f32"]
pert = (f64[:, 0] & 2) > 0
same = (f64[:, 0] == f32[:, 0])
print("first step: pert", pert.sum(), "same flags", same.mean())
x, y = a64[pert, 0], a32[pert, 0]
print("mean a f64", x.mean(), "f32", y.mean())
d = np.abs(x - y)
idx = np.argsort(-d)[:15]
for i in idx: print(f"a64={x[i]:.6f} a32={y[i]:.6f}")
print("fraction a32==0 where a64>0.5:", np.mean((y == 0) & (x > 0.5)), "a64==0 where a32>0.5:", np.mean((x == 0) & (y > 0.5)))

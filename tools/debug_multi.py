"""Debug: single handle (coop / per-step) vs multi-device handle, Global mirror."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2402_08273_b200 import Engine, RenderConfig, scenes

scene = scenes.mirror_box()
C = 301
strategy = sys.argv[1] if len(sys.argv) > 1 else "global"
kw = dict(strategy=strategy, perturbation="lens", chains=C, mutations=C * 24 + 17, m_refine=C * 5 + 50, m_split=40,
          n_top=4, n_bottom=3, metrics_interval=C * 7 + 3, width=40, height=40, max_vertices=12, b_samples=3000,
          seed=21, precision="f64", rng="philox", log_steps=24, adapt_mode="pooled", trace_enabled=True)


def run(devices=None, coop=True, film=3):
    if coop:
        os.environ.pop("RAMLT_COOP", None)
    else:
        os.environ["RAMLT_COOP"] = "0"
    e = Engine(scene, RenderConfig(**kw), devices=devices, film_sync_steps=film)
    e.set_b(1.7)
    e.init_chains()
    e.run(kw["mutations"])
    a, f = e.decisions(24)
    tr = e.trace()
    e.close()
    return f, tr


ref_f, ref_tr = run()
for name, args in [("single per-step", dict(coop=False)), ("multi [0,0] film3", dict(devices=[0, 0])),
                   ("multi [0,0] nofilm", dict(devices=[0, 0], film=0)), ("multi [0] ", dict(devices=[0]))]:
    f, tr = run(**args)
    d = np.argwhere(f != ref_f)
    print(name, "flags equal" if d.size == 0 else f"first flag diffs {d[:4].tolist()}")
    n = min(len(tr), len(ref_tr))
    bad = np.flatnonzero(np.any(tr[:n] != ref_tr[:n], axis=1))
    print("   trace rows", len(tr), len(ref_tr), "first diff", bad[:1].tolist(),
          tr[bad[0]].tolist() if bad.size else "", ref_tr[bad[0]].tolist() if bad.size else "")

"""Quick throughput probe of the engine (not the bench contract; see bench.py)."""
import sys
import time

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))

from paper_2402_08273_b200 import Engine, RenderConfig, scenes  # noqa: E402


def probe(scene_name, strategy, perturbation, chains, steps, lanes, precision="f32", rng="philox",
          maxv=9, res=256, spl=0):
    scene = scenes.SCENES[scene_name]()
    cfg = RenderConfig(strategy=strategy, perturbation=perturbation, chains=chains,
                       mutations=chains * steps, width=res, height=res, max_vertices=maxv,
                       b_samples=100000, precision=precision, rng=rng, lanes_per_chain=lanes,
                       metrics_interval=chains * steps, m_refine=10_000_000 // chains * chains,
                       steps_per_launch=spl)
    eng = Engine(scene, cfg)
    t = time.time()
    eng.estimate_b()
    eng.init_chains()
    eng.synchronize()
    t1 = time.time()
    eng.run(chains * 8)   # warm-up
    eng.synchronize()
    t2 = time.time()
    eng.run(chains * steps)
    eng.synchronize()
    t3 = time.time()
    s = eng.stats()
    m = chains * steps
    print(f"{scene_name:8s} {strategy:12s} {perturbation:11s} C={chains:7d} G={lanes:2d} {precision} {rng}: "
          f"prologue {t1 - t:.2f}s  {m / (t3 - t2) / 1e6:9.2f} M mut/s  acc={s.mean_acceptance:.3f} "
          f"rays/mut={(s.rays_closest + s.rays_visibility) / max(s.total_mutations, 1):.2f} "
          f"launches={s.kernel_launches}", flush=True)
    eng.close()


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("all", "lanes"):
        for g in (1, 2, 4):
            probe("caustic", "ra-quadtree", "multi-chain", 262144, 16, g, maxv=17, res=512)
            probe("cornell", "fixed", "lens", 262144, 16, g)
    if which in ("all",):
        probe("cornell", "fixed", "lens", 1024, 512, 32)
        probe("cornell", "fixed", "lens", 1024, 512, 16)
        probe("cornell", "ra-quadtree", "lens", 1024, 512, 32)
        probe("caustic", "fixed", "multi-chain", 262144, 16, 1, maxv=17, res=512)
        probe("cornell", "fixed", "lens", 1024, 128, 32, precision="f64", rng="pcg32")


def probe_c4(chains=1 << 20, steps=8, strategy="ra-quadtree", n_tris=1 << 20, accel="auto"):
    t0 = time.time()
    text = scenes.cluster_room(n_tris=n_tris)
    t1 = time.time()
    cfg = RenderConfig(strategy=strategy, perturbation="lens", chains=chains, mutations=chains * steps,
                       width=1024, height=1024, max_vertices=13, b_samples=100000, precision="f32",
                       rng="philox", metrics_interval=chains * steps, accel=accel)
    eng = Engine(text, cfg)
    t2 = time.time()
    eng.estimate_b()
    eng.init_chains()
    eng.synchronize()
    t3 = time.time()
    eng.run(chains * 2)
    eng.synchronize()
    t4 = time.time()
    eng.run(chains * steps)
    eng.synchronize()
    t5 = time.time()
    s = eng.stats()
    print(f"c4 {strategy} C={chains} tris={n_tris} accel={accel}: gen {t1-t0:.1f}s create(parse+bvh) {t2-t1:.1f}s "
          f"b+init {t3-t2:.2f}s  {chains*steps/(t5-t4)/1e6:.2f} M mut/s acc={s.mean_acceptance:.3f} "
          f"rays/mut={(s.rays_closest + s.rays_visibility) / max(s.total_mutations, 1):.2f}", flush=True)
    eng.close()


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "c4":
    probe_c4()
    probe_c4(strategy="fixed")

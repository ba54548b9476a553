"""Phase breakdown of the bench's end-to-end path (parse, create incl. BVH,
estimate_b, chain init, steps, image readback) for one workload."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2402_08273_b200 import Engine, RenderConfig, parse_scene, scenes  # noqa: E402


def main(name="c5", steps=16):
    steps = int(steps)
    wl = bench.WORKLOADS[name]
    t = [time.perf_counter()]
    text = scenes.SCENES[wl["scene"]](**wl["scene_args"])
    t.append(time.perf_counter())
    sc = parse_scene(text)
    t.append(time.perf_counter())
    Cn = wl["chains"]
    cfg = RenderConfig(strategy=wl["strategy"], perturbation=wl["perturbation"], chains=Cn,
                       mutations=Cn * steps, width=wl["width"], height=wl["height"],
                       max_vertices=wl["max_vertices"], b_samples=1_000_000, seed=2,
                       precision="f32", rng="philox", metrics_interval=Cn * steps)
    eng = Engine(sc, cfg)
    eng.synchronize()
    t.append(time.perf_counter())
    eng.estimate_b()
    eng.synchronize()
    t.append(time.perf_counter())
    eng.init_chains()
    eng.synchronize()
    t.append(time.perf_counter())
    eng.run(Cn * steps)
    eng.synchronize()
    t.append(time.perf_counter())
    eng.image()
    t.append(time.perf_counter())
    names = ["gen text", "parse", "create(+bvh)", "estimate_b", "init", f"{steps} steps", "image"]
    print(name, " ".join(f"{n}={b - a:.3f}s" for n, a, b in zip(names, t, t[1:])), flush=True)


if __name__ == "__main__":
    main(*(sys.argv[1:3] or ["c5"]))

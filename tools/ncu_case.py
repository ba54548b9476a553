"""Small single-config run for ncu captures: python tools/ncu_case.py <scene> <strategy> <pert> <chains> <steps> [maxv] [res]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_08273_b200 import Engine, RenderConfig, scenes
scene, strat, pert, C, steps = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
maxv = int(sys.argv[6]) if len(sys.argv) > 6 else 17
res = int(sys.argv[7]) if len(sys.argv) > 7 else 512
cfg = RenderConfig(strategy=strat, perturbation=pert, chains=C, mutations=C * steps, width=res, height=res,
                   max_vertices=maxv, b_samples=65536, precision="f32", rng="philox",
                   metrics_interval=C * steps, steps_per_launch=int(os.environ.get("SPL", "0")))
kw = {"n_tris": int(os.environ["NTRIS"])} if os.environ.get("NTRIS") else {}
eng = Engine(scenes.SCENES[scene](**kw), cfg)
eng.estimate_b(); eng.init_chains(); eng.run(C * steps); eng.synchronize()
s = eng.stats()
print("ok", s.total_mutations, s.kernel_launches)

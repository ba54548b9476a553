"""A/B throughput of library variants on the benched configuration (steady state):
python tools/ab.py [c5|c4|c3] lib1 lib2 ...   (lib = "" for _lib/libramlt_gpu.so, else the
variant name built by tools/build_variants.sh).  Each variant runs in its own process,
twice, interleaved; burn-in 12 steps, then 12 timed steps (CUDA events)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = {"c5": dict(scene="clusters", chains=1 << 23, res=2048, maxv=13, strategy="ra-quadtree", pert="lens"),
         "c4": dict(scene="clusters", chains=1 << 20, res=1024, maxv=13, strategy="ra-quadtree", pert="lens"),
         "c3": dict(scene="caustic", chains=262144, res=512, maxv=17, strategy="ra-quadtree", pert="multi-chain")}

CHILD = r'''
import sys, os
sys.path.insert(0, ROOT)
import torch
from paper_2402_08273_b200 import Engine, RenderConfig, scenes
c = CASE
text = scenes.SCENES[c["scene"]]()
C = c["chains"]
eng = Engine(text, RenderConfig(strategy=c["strategy"], perturbation=c["pert"], chains=C, mutations=C * 4096,
             width=c["res"], height=c["res"], max_vertices=c["maxv"], b_samples=100000, precision="f32",
             rng="philox", metrics_interval=C * 4096,
             m_refine=int(os.environ.get("M_REFINE", "0")) or max(1, round(1e7 / C)) * C, lanes_per_chain=int(os.environ.get("LANES", "0"))))
s = torch.cuda.current_stream()
eng.set_stream(s.cuda_stream)
eng.estimate_b(); eng.init_chains()
eng.run(C * 12)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s); eng.run(C * 12); e1.record(s); torch.cuda.synchronize()
st = eng.stats()
print("RESULT %.2f" % (C * 12 / (e0.elapsed_time(e1) / 1e3) / 1e6), "acc %.3f" % st.mean_acceptance, flush=True)
'''

case = sys.argv[1]
libs = sys.argv[2:] or [""]
res = {l: [] for l in libs}
for rep in range(2):
    for l in libs:
        env = dict(os.environ)
        lib, _, envs = l.partition("@")   # "variant@VAR=1,VAR2=3": library variant and/or env settings
        if lib:
            env["RAMLT_GPU_LIB"] = os.path.join(ROOT, "paper_2402_08273_b200", "_lib", f"libramlt_gpu_{lib}.so")
        for kv in filter(None, envs.split(",")):
            k, _, v = kv.partition("=")
            env[k] = v
        code = CHILD.replace("ROOT", repr(ROOT)).replace("CASE", repr(CASES[case]))
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        line = [x for x in out.stdout.splitlines() if x.startswith("RESULT")]
        res[l].append(float(line[0].split()[1]) if line else float("nan"))
        print(f"{case} {l or 'default':12s} rep{rep}: {line[0] if line else out.stderr[-400:]}", flush=True)
for l in libs:
    print(f"{case} {l or 'default':12s} mean {sum(res[l]) / len(res[l]):.2f} M mut/s")

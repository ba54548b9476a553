"""Benchmark of the B200 MLT hot path (contract: see DESIGN.md §6).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3|c1] [--impl ours|reference]

One "step" = one lockstep mutation of every chain (C mutations).  Rank 0 prints
ONE JSON line.  Under torchrun (N > 1) chains shard across ranks
(paper_2402_08273_b200.distributed); timing is CUDA events on the engine's
stream, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs; "strategy/perturbation" follow the
# reference defaults (RA-quadtree) and the survey's per-config perturbation.
WORKLOADS = {
    "c3": dict(scene="caustic", scene_args={}, chains=262144, steps_per_chain=1 << 16, width=512,
               height=512, max_vertices=17, strategy="ra-quadtree", perturbation="multi-chain",
               bound="fp32", scaling="weak", e2e_steps=256, cpu_sample=1 << 21, cpu_b=4096,
               desc="C3 caustic box: 36 tri + glass sphere, 1% light, 512^2, path length 16, "
                    "262,144 chains"),
    "c1": dict(scene="cornell", scene_args={}, chains=1024, steps_per_chain=1 << 20, width=256,
               height=256, max_vertices=9, strategy="ra-quadtree", perturbation="lens",
               bound="fp32", scaling="weak", e2e_steps=256, cpu_sample=1 << 21, cpu_b=4096,
               desc="C1 Cornell box: 36 tri, 256^2, path length 8, 1,024 chains"),
    "c4": dict(scene="clusters", scene_args={"n_tris": 1 << 20}, chains=1 << 20, steps_per_chain=1 << 12,
               width=1024, height=1024, max_vertices=13, strategy="ra-quadtree", perturbation="lens",
               bound="hbm", scaling="weak", e2e_steps=128, cpu_sample=256, cpu_b=16,
               desc="C4 clustered room: 2^20 + 20 tri (64 clusters, 4 lights), 1024^2, path length 12, "
                    "1,048,576 chains, SAH BVH"),
    "c5": dict(scene="clusters", scene_args={"n_tris": 1 << 20}, chains=1 << 23, steps_per_chain=1 << 12,
               width=2048, height=2048, max_vertices=13, strategy="ra-quadtree", perturbation="lens",
               bound="hbm", scaling="strong", e2e_steps=128, cpu_sample=256, cpu_b=16,
               desc="C5 scaling config: the C4 scene at 2048^2, 8,388,608 chains split across the GPUs"),
}
# configs[1]: the analytic-target adaptive MCMC harness (include/ramlt_mix.h);
# a parity case of the metric's family, measured on its own line (not the default)
C2 = dict(chains=65536, steps=4096, dim=8, n_comp=4, target_seed=0, strategy="global",
          desc="C2 analytic target: 4 anisotropic Gaussians in [0,1]^8, 65,536 chains x 4,096 steps, "
               "Global (scalar lambda) pooled adaptation")


def m_refine_for(chains: int) -> int:
    """The paper's M_refine = 10^7 global mutations (core/driver.hpp:30), rounded to the
    nearest multiple of the chain count so that every span is a whole number of lockstep
    steps and every chain takes the same number of steps (SURVEY.md §8 C1 rule; the raw
    10^7 splits each span of 8,388,608 chains into a full and a 19 % lockstep step)."""
    return max(1, round(10_000_000 / chains)) * chains


METRIC = "MLT mutations/sec"
UNIT = "mutations/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max(float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[2:]) if v.strip() == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def reference_rays_per_mutation(wl: dict, scene_text: str, threads: int):
    """R_m: reference ray casts (closest-hit + visibility) per mutation, counted
    by the UNMODIFIED reference on the benched scene itself (oracle/_ref
    libramlt_ref_log.so: link-time --wrap counters on SceneModel::intersect /
    visible, counted inside the mutation loop only), with
    chains = host threads.  Falls back to the restatement oracle when the
    reference was not built."""
    from oracle.abi import OracleConfig, OracleLib, RefLib, REF_LOG_SO
    big = wl["scene"] == "clusters"
    per = 32 if big else 256
    cfg = OracleConfig(strategy=wl["strategy"], perturbation=wl["perturbation"], chains=threads,
                       mutations=threads * per, width=wl["width"], height=wl["height"],
                       max_vertices=wl["max_vertices"], b_samples=16 if big else 4096, seed=3,
                       metrics_interval=threads * per)
    if os.path.exists(REF_LOG_SO):
        o = RefLib(log=True).render(scene_text, cfg, log_steps=1)
        src = (f"counted by the unmodified reference on the benched scene ({threads} threads x {per} "
               f"mutations, loop-only --wrap counters)")
    else:
        cfg.chains, cfg.mutations = 8, 8 * per
        o = OracleLib().render(scene_text, cfg, log_steps=1)
        src = f"counted by the restatement oracle on the benched scene (8 chains x {per} mutations)"
    return (o.stats.rays_closest + o.stats.rays_visibility) / max(o.stats.total_mutations, 1), src


def relmse_vs_reference(args):
    """relMSE vs CPU (BASELINE.json metric): the f32 engine against the
    unmodified reference at EQUAL mutation counts on a configuration the
    reference can run as specified -- C1 (Cornell box, 1,024 chains, 256^2,
    path length 8, RA-quadtree lens).  error_report rRMSE (core/diagnostics.cpp:
    11-38, eps 1e-2, luminance) of the GPU image against reference seed 1,
    next to the reference's own seed-to-seed rRMSE (seed 2 vs seed 1) measured
    in the same run; tolerance 1.5x that noise."""
    import numpy as np
    from oracle.abi import OracleConfig, RefLib, REF_SO, ref_error_report
    from paper_2402_08273_b200 import Engine, RenderConfig, scenes
    if not os.path.exists(REF_SO):
        return {"unavailable": "oracle/_ref not built"}
    text = scenes.cornell_box()
    wl = WORKLOADS["c1"]
    M = args.relmse_mutations
    common = dict(strategy=wl["strategy"], perturbation=wl["perturbation"], chains=wl["chains"], mutations=M,
                  width=wl["width"], height=wl["height"], max_vertices=wl["max_vertices"], b_samples=1_000_000,
                  metrics_interval=M)
    lib = RefLib(log=False)
    t0 = time.perf_counter()
    r1 = lib.render(text, OracleConfig(**common, seed=1))
    r2 = lib.render(text, OracleConfig(**common, seed=2))
    t_ref = time.perf_counter() - t0
    eng = Engine(text, RenderConfig(**common, seed=3, precision="f32", rng="philox"))
    eng.set_reference(r1.image)
    eng.render()
    err = eng.rrmse(M)            # the engine's own error_report (k_rrmse_partial) against the reference image
    s = eng.stats()
    eng.close()
    noise = ref_error_report(lib, r2.image, r1.image)
    return {"value": err, "noise": noise, "tolerance": 1.5 * noise, "ratio": err / noise,
            "pass": bool(err <= 1.5 * noise),
            "acceptance": {"gpu": s.mean_acceptance, "reference_seed1": r1.stats.mean_acceptance,
                           "reference_seed2": r2.stats.mean_acceptance},
            "b": {"gpu": s.b, "reference": r1.stats.b},
            "config": (f"C1 Cornell box, {wl['chains']} chains, {wl['width']}^2, max_vertices {wl['max_vertices']}, "
                       f"{wl['strategy']} {wl['perturbation']}, {M} mutations each; GPU f32/Philox vs the "
                       f"unmodified reference (seeds 1, 2; {wl['chains']} threads, {t_ref:.1f} s)"),
            "metric": "error_report rRMSE (luminance, eps 1e-2) vs reference seed 1"}


def cpu_reference_run(wl: dict, scene_text: str, mutations: int, threads: int):
    """The reference's own run_render (oracle/_ref, unmodified sources) on host
    cores: chains = threads (one std::thread per chain, core/driver.cpp:282-297).
    Falls back to the restatement oracle (single thread) when the reference
    library was not built."""
    from oracle.abi import OracleConfig, RefLib, OracleLib, REF_SO
    cfg = OracleConfig(strategy=wl["strategy"], perturbation=wl["perturbation"], chains=threads,
                       mutations=mutations, width=wl["width"], height=wl["height"],
                       max_vertices=wl["max_vertices"], b_samples=wl.get("cpu_b", 4096), seed=1,
                       metrics_interval=mutations, m_refine=10_000_000)
    if os.path.exists(REF_SO):
        out = RefLib(log=False).render(scene_text, cfg)
        kind, cores = "reference", threads
    else:
        cfg.chains = 1
        out = OracleLib().render(scene_text, cfg)
        kind, cores = "port", 1
    t = out.stats.loop_time_s
    return out.stats.total_mutations / t, kind, cores, t, cfg.chains


def _acc_sums(eng):
    """(accepted-probability sum, perturbation proposals) of this rank so far."""
    s = eng.stats()
    return s.mean_acceptance * s.perturbation_proposals, float(s.perturbation_proposals)


def run_ours(args, wl, scene_text):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2402_08273_b200 import Engine, RenderConfig
    from paper_2402_08273_b200.distributed import ShardPlan, ShardedRender

    world, rank, local = dist_env()
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        # RAMLT_DIST_BACKEND=gloo runs the same N > 1 code path with ranks sharing
        # a GPU (functional check on a 1-GPU box); production is NCCL.
        backend = os.environ.get("RAMLT_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    C = wl["chains"]
    plan = ShardPlan(C, world, rank)
    stream = torch.cuda.current_stream()
    cfg = RenderConfig(strategy=wl["strategy"], perturbation=wl["perturbation"], chains=C,
                       mutations=C * wl["steps_per_chain"], width=wl["width"], height=wl["height"],
                       max_vertices=wl["max_vertices"], b_samples=1_000_000, seed=1,
                       precision="f32", rng="philox", device=local, profile_kernels=True,
                       metrics_interval=C * wl["steps_per_chain"], m_refine=m_refine_for(C))
    # one process per GPU: chains shard by global id; pooled adaptation exchanged
    # every lockstep step, quadtree visits at every refine barrier, the film every
    # 2^12 lockstep steps (configs[4]) -- distributed.ShardedRender
    sr = ShardedRender(wl["scene_text"], cfg, exchange_every=1, film_sync_steps=4096)
    eng = sr.engine
    sr.estimate_b()
    sr.init_chains()

    def step():
        sr.run(C)

    def window_acceptance(a0, n0):
        a1, n1 = _acc_sums(eng)
        t = torch.tensor([a1 - a0, n1 - n0], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t[0] / t[1]) if t[1] > 0 else 0.0, (a1, n1)

    # burn-in (outside the timed region): the adaptive controller starts at
    # lambda_init = 1 (sigma = e^0.5 rad) far from alpha* = 0.5; step until the
    # pooled window acceptance is within 0.1 of the target (steady state), at
    # most burnin_max steps.  Fixed strategies need none.
    burn, burn_acc = 0, None
    sums = _acc_sums(eng)
    if cfg.strategy != "fixed":
        target = cfg.target_acceptance
        while burn < args.burnin_max:
            step()
            burn += 1
            burn_acc, sums = window_acceptance(*sums)
            if burn >= 4 and abs(burn_acc - target) <= 0.1:
                break
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    sums = _acc_sums(eng)
    s0 = eng.stats()
    d0 = sr.done
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        if world > 1:
            for _ in range(args.steps):
                step()
        else:
            # one call: the engine batches the lockstep steps of a span itself
            # (cooperative launches for adaptive runs with few chains)
            sr.run(C * args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        dist.barrier()
    s1 = eng.stats()
    acc_window, _ = window_acceptance(*sums)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    muts = sr.done - d0   # = steps x C (N > 1: whole lockstep steps of the canonical spans)
    value = muts / (ms_max / 1e3)
    launches = s1.kernel_launches - s0.kernel_launches
    step_ms = (s1.step_kernel_ms - s0.step_kernel_ms)
    step_launches = s1.step_kernel_launches - s0.step_kernel_launches
    trace_ms = s1.trace_kernel_ms - s0.trace_kernel_ms
    trace_launches = s1.trace_kernel_launches - s0.trace_kernel_launches
    wf_rounds = s1.wavefront_rounds - s0.wavefront_rounds
    rays_dev = (s1.rays_closest + s1.rays_visibility) - (s0.rays_closest + s0.rays_visibility)
    rays_t = torch.tensor([float(rays_dev)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(rays_t, op=dist.ReduceOp.SUM)
    k = eng.chain_lengths()
    k_bar = float(k.mean()) if k.size else float("nan")
    ceiling = None
    if wl["scene"] == "clusters" and rank == 0:
        # the traversal-only ceiling of this BVH (k_trace_bench: the step kernel's
        # traversal loop on incoherent closest-hit rays), measured after the timed region
        eng.trace_benchmark(1 << 22)
        n_rays = 1 << 26
        tms, _ = eng.trace_benchmark(n_rays)
        ceiling = n_rays / (tms / 1e3)
    eng.close()
    return dict(value=value, ms=ms_max, launches=launches, step_ms=step_ms,
                step_launches=step_launches, trace_ms=trace_ms, trace_launches=trace_launches,
                wf_rounds=wf_rounds, rays_local=float(rays_dev), rays_dev=float(rays_t.item()), muts=muts, clocks=clk.summary(),
                world=world, rank=rank, local=local, mutations_per_rank=muts * plan.count / C,
                acceptance=acc_window, burnin=dict(steps=burn, acceptance=burn_acc, max=args.burnin_max),
                k_bar=k_bar, ceiling=ceiling)


def run_e2e(args, wl):
    """End to end through the reference-facing C-ABI with host buffers: scene
    text from host memory -> ramlt_gpu_create_from_text -> ramlt_gpu_render
    (estimate_b, chain init, K steps) -> ramlt_gpu_read_image into a host array."""
    import ctypes as C
    import numpy as np
    import torch
    from paper_2402_08273_b200 import _capi
    from paper_2402_08273_b200.render import RenderConfig
    lib = _capi.load()
    Cn = wl["chains"]
    steps = max(args.steps, wl["e2e_steps"])
    cfg = RenderConfig(strategy=wl["strategy"], perturbation=wl["perturbation"], chains=Cn,
                       mutations=Cn * steps, width=wl["width"], height=wl["height"],
                       max_vertices=wl["max_vertices"], b_samples=1_000_000, seed=2,
                       precision="f32", rng="philox", device=0,
                       metrics_interval=Cn * steps, m_refine=m_refine_for(Cn))
    text = wl["scene_text"].encode()
    img = np.zeros((wl["height"], wl["width"], 3), np.float32)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = C.c_void_p()
    d = cfg.to_c()
    rc = lib.ramlt_gpu_create_from_text(text, b"<bench>", C.byref(d), C.byref(h))
    assert rc == 0, lib.ramlt_gpu_last_create_error()
    rc = lib.ramlt_gpu_render(h)
    assert rc == 0, lib.ramlt_gpu_last_error(h)
    rc = lib.ramlt_gpu_read_image(h, img.ctypes.data_as(C.POINTER(C.c_float)))
    assert rc == 0
    t1 = time.perf_counter()
    lib.ramlt_gpu_destroy(h)
    return Cn * steps / (t1 - t0), len(text), img.nbytes, float(img.mean())


def run_e2e_sharded(args, wl):
    """N > 1 end to end through the public sharded API
    (paper_2402_08273_b200.distributed.ShardedRender): scene text from host
    memory, per-rank create, gathered b, init, K lockstep steps with the pooled
    adaptation exchange, film SUM all-reduce, rank 0 copies the film to the host.
    Wall clock, max over ranks."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2402_08273_b200.distributed import ShardedRender
    from paper_2402_08273_b200.render import RenderConfig
    Cn = wl["chains"]
    steps = max(args.steps, wl["e2e_steps"])
    cfg = RenderConfig(strategy=wl["strategy"], perturbation=wl["perturbation"], chains=Cn,
                       mutations=Cn * steps, width=wl["width"], height=wl["height"],
                       max_vertices=wl["max_vertices"], b_samples=1_000_000, seed=2,
                       precision="f32", rng="philox", metrics_interval=Cn * steps, m_refine=m_refine_for(Cn))
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sr = ShardedRender(wl["scene_text"], cfg)
    film = sr.render()
    host = film.cpu().numpy() if dist.get_rank() == 0 else None
    torch.cuda.synchronize()
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64,
                     device=torch.device("cuda", torch.cuda.current_device()))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    sr.engine.close()
    nbytes = host.nbytes if host is not None else 0
    return Cn * steps / float(t.item()), len(wl["scene_text"]), nbytes, 0.0


def c2_flop_per_step(D: int, K: int) -> float:
    """Algorithmic FP32 work of one chain step: K components x
    (D sub + D(D+1)/2 mul + D(D-1)/2 add + 2D for |z|^2 + 2) + logsumexp (2K+1)
    + D proposals x (Acklam central branch 24 + 2) + the MH ratio (2)."""
    return K * (D * D + 3 * D + 2) + (2 * K + 1) + 26 * D + 2


def bench_c2(args):
    """configs[1] line: device-resident timing of K lockstep steps of all
    chains (one cooperative launch per 1,024 steps), plus the e2e run through
    the C-ABI with host buffers and the reference-composition CPU baseline."""
    import ctypes as C
    import numpy as np
    import torch
    from paper_2402_08273_b200 import _capi
    from paper_2402_08273_b200.mix import MixConfig, MixEngine, MixTarget
    world, rank, local = dist_env()
    steps = args.steps
    config = {"workload": "c2", "desc": C2["desc"], "chains": C2["chains"], "dim": C2["dim"],
              "n_comp": C2["n_comp"], "strategy": C2["strategy"], "adaptation": "pooled",
              "step": "one lockstep step (propose, evaluate, accept, adapt) of every chain",
              "l2": "chain state (2.6 MB) is L2-resident by design: the kernel keeps chains in registers "
                    "across steps, so no flush applies", "rng": "philox4x32-10"}
    tgt = MixTarget.config2(C2["target_seed"], C2["dim"], C2["n_comp"])
    D, K = C2["dim"], C2["n_comp"]
    threads = os.cpu_count() or 1
    if args.impl == "reference":
        if rank != 0:
            return
        line = c2_cpu_line(args, tgt, config)
        print(json.dumps(line), flush=True)
        return
    if world > 1:
        raise SystemExit("c2 is a single-GPU parity workload (replicas only); run it with --gpus 1")
    torch.cuda.set_device(local)
    stream = torch.cuda.current_stream()
    eng = MixEngine(tgt, MixConfig(strategy=C2["strategy"], chains=C2["chains"], seed=1, precision="f32",
                                   rng="philox", adapt_mode="pooled", device=local, profile_kernels=True))
    eng.set_stream(stream.cuda_stream)
    eng.init_chains()
    eng.run(args.warmup)
    torch.cuda.synchronize()
    s0 = eng.stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        eng.run(steps)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    s1 = eng.stats()
    muts = steps * C2["chains"]
    value = muts / (ms / 1e3)
    launches = s1.kernel_launches - s0.kernel_launches
    kms = s1.step_kernel_ms - s0.step_kernel_ms
    kl = max(s1.step_kernel_launches - s0.step_kernel_launches, 1)
    acc = s1.mean_acceptance
    eng.close()
    w = c2_flop_per_step(D, K)
    sm_max = clk.summary().get("sm_max_mhz") or 1965.0
    peak = 148 * 128 * 2 * float(sm_max) * 1e6 / 1e12
    achieved = (muts / kl) * w / ((kms / kl) / 1e3) / 1e12
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic_c2.json"))).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        traffic = None
    roofline = {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "peak_source": "nominal FP32 issue: 148 SM x 128 lanes x 2 x sm_max_mhz",
                "work_per_unit": f"{w:.0f} FLOP per chain step (K(D^2+3D+2) + 2K+1 + 26D + 2, D={D}, K={K})",
                "kernel": "k_mix_coop (persistent cooperative chain-step kernel)",
                "kernel_share": kms / ms if ms else None}
    # e2e through the C-ABI: host target arrays -> create/init/run -> host states
    lib = _capi.load()
    t_c, keep = tgt.to_c()
    d = MixConfig(strategy=C2["strategy"], chains=C2["chains"], seed=2, precision="f32", rng="philox",
                  adapt_mode="pooled", device=local).to_c()
    xs = np.zeros((C2["chains"], D))
    lps = np.zeros(C2["chains"])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = C.c_void_p()
    assert lib.ramlt_mix_create(C.byref(t_c), C.byref(d), C.byref(h)) == 0
    assert lib.ramlt_mix_init_chains(h) == 0
    assert lib.ramlt_mix_run(h, steps) == 0
    dp = C.POINTER(C.c_double)
    assert lib.ramlt_mix_read_state(h, xs.ctypes.data_as(dp), lps.ctypes.data_as(dp)) == 0
    t1 = time.perf_counter()
    lib.ramlt_mix_destroy(h)
    h2d = sum(a.nbytes for a in keep)
    cpu = None
    if not args.no_cpu_baseline:
        ref = c2_cpu_line(args, tgt, config)
        cpu = ref["cpu_baseline"]
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": steps,
            "warmup": args.warmup, "ms_per_step": ms / steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded configs[1] target)", "config": config,
            "mean_acceptance": acc, "roofline": roofline, "cpu_baseline": cpu,
            "e2e": {"value": muts / (t1 - t0), "unit": UNIT, "h2d_bytes_per_step": h2d / steps,
                    "d2h_bytes_per_step": (xs.nbytes + lps.nbytes) / steps, "steps": steps,
                    "path": "ramlt_mix_create (host target) + init + run(K) + ramlt_mix_read_state, wall clock"},
            "gpu_launches": launches, "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


def c2_cpu_line(args, tgt, config):
    """The reference composition (oracle/_ref ref_mix_run: the reference's
    controller, mh_accept, normal_quantile and PCG32) on one host thread, on a
    bounded sample: 256 chains x 256 steps per measurement."""
    from oracle.abi import OracleMixConfig, REF_SO, mix_run
    reference = os.path.exists(REF_SO)
    chains, steps = 256, 256
    vals = []
    for _ in range(min(max(args.steps // 512, 1), 4)):
        t0 = time.perf_counter()
        mix_run(tgt, OracleMixConfig(strategy=C2["strategy"], chains=chains, steps=steps, seed=1,
                                     rng="pcg32", adapt_mode="literal"), reference=reference)
        vals.append(chains * steps / (time.perf_counter() - t0))
    v = sum(vals) / len(vals)
    cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "reference" if reference else "port",
           "sample": f"{chains} chains x {steps} lockstep steps of the c2 target, one host thread "
                     f"(the reference's controller / accept / quantile / PCG32 composition)"}
    return {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": 0, "steps": len(vals), "warmup": 0,
            "ms_per_step": 1e3 * chains * steps / v, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded configs[1] target)",
            "impl": "reference", "config": dict(config, chains_cpu=chains), "cpu_baseline": cpu,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default 16; c2: 4096)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c5", choices=sorted(WORKLOADS) + ["c2"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=0, help="mutations in the CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-relmse", action="store_true", help="skip the relMSE-vs-reference leg (C1)")
    ap.add_argument("--relmse-mutations", type=int, default=1 << 24)
    ap.add_argument("--burnin-max", type=int, default=64,
                    help="max untimed burn-in steps until the window acceptance is within 0.1 of the target")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.steps is None:
        args.steps = C2["steps"] if args.workload == "c2" else 16
    if args.workload == "c2":
        bench_c2(args)
        return

    from paper_2402_08273_b200 import scenes
    wl = dict(WORKLOADS[args.workload])
    wl["scene_text"] = scenes.SCENES[wl["scene"]](**wl["scene_args"])
    world, rank, local = dist_env()
    threads = os.cpu_count() or 1
    config = {"workload": args.workload, "desc": wl["desc"], "chains": wl["chains"],
              "strategy": wl["strategy"], "perturbation": wl["perturbation"],
              "image": [wl["width"], wl["height"]], "max_vertices": wl["max_vertices"],
              "step": "one lockstep mutation of every chain",
              "l2": "inputs larger than the 126 MB L2, no flush (chain path SoA: c3 134 MB, c4 400 MB, "
                    "c5 3.2 GB; c4/c5 BVH + triangles ~120 MB)",
              "rng": "philox4x32-10", "adaptation": "pooled" if wl["chains"] > 4096 else "literal",
              "m_refine": m_refine_for(wl["chains"]),
              "m_refine_note": "the multiple of the chain count nearest the paper's 10^7 (whole lockstep steps per span)"}

    if args.impl == "reference":
        if rank != 0:
            return
        sample = args.cpu_sample or wl["cpu_sample"]
        vals, times = [], []
        n_warm = args.warmup if args.warmup < 3 else 1
        for _ in range(n_warm):
            cpu_reference_run(wl, wl["scene_text"], max(sample // 8, threads), threads)
        for _ in range(min(args.steps, 8 if wl["bound"] == "fp32" else 2)):
            v, kind, cores, t, chains = cpu_reference_run(wl, wl["scene_text"], sample, threads)
            vals.append(v)
            times.append(t)
        v = sum(vals) / len(vals)
        line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": 0, "steps": len(vals),
                "warmup": n_warm, "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
                "scaling": wl["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "impl": "reference", "config": dict(config, chains_cpu=chains),
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                                 "sample": f"{sample} mutations of the {args.workload} scene/variant "
                                           f"with chains = {chains} host threads"},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    res = run_ours(args, wl, wl["scene_text"])
    if res["world"] > 1:
        res["e2e"] = run_e2e_sharded(args, wl)
    if res["rank"] != 0:
        return
    peaks = load_peaks()
    threads = os.cpu_count() or 1
    r_m, r_m_src = reference_rays_per_mutation(wl, wl["scene_text"], threads)
    from paper_2402_08273_b200 import parse_scene
    n_mat, n_sph, n_tri, n_emi = parse_scene(wl["scene_text"]).counts
    flop_per_mut = r_m * (45.0 * n_tri + 20.0 * n_sph)
    # dominant kernel: the chain-step kernel; algorithmic work per launch
    # = mutations per launch (all chains of this rank) x W, / its mean event time
    per_launch_muts = res["mutations_per_rank"] / max(res["step_launches"], 1)
    mean_launch_s = (res["step_ms"] / max(res["step_launches"], 1)) / 1e3
    achieved = per_launch_muts * flop_per_mut / mean_launch_s / 1e12
    sm_max = res["clocks"].get("sm_max_mhz") or peaks.get("sm_max_mhz", 1965.0)
    fp32_peak = 148 * 128 * 2 * float(sm_max) * 1e6 / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.workload}.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            traffic = tj.get("dram_bytes_per_launch")
            if "dram_bytes_per_mutation" in tj:   # launches of this workload vary in size
                traffic = tj["dram_bytes_per_mutation"] * per_launch_muts
        except Exception:
            traffic = None
    if wl["bound"] == "fp32":
        roofline = {"bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                    "frac": achieved / fp32_peak, "traffic": traffic,
                    "peak_source": "nominal FP32 issue: 148 SM x 128 lanes x 2 x sm_max_mhz "
                                   "(MEASURED_PEAKS.json has no FP32 figure)",
                    "work_per_unit": f"R_m x (45 N_tri + 20 N_sph) = {r_m:.3f} x (45x{n_tri} + 20x{n_sph}) "
                                     f"= {flop_per_mut:.0f} FLOP/mutation (R_m: {r_m_src})"}
    else:
        # B = R_m x B_ray + B_state per mutation, B_ray = one
        # BVH root-to-leaf descent (64 B per level) + 4 triangles x 48 B
        import math
        levels = max(1, math.ceil(math.log2(max(n_tri / 4.0, 2.0))))
        b_ray = 64.0 * levels + 4 * 48.0
        k_bar = res["k_bar"]   # measured: mean current path length over all chains after the timed steps
        b_state = 2.0 * (16.0 * k_bar + 48.0) + 32.0
        bytes_per_mut = r_m * b_ray + b_state
        ach = per_launch_muts * bytes_per_mut / mean_launch_s / 1e9
        peak = float(peaks.get("hbm_gbs", 6650.0))
        roofline = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                    "traffic": traffic,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650 GB/s",
                    "work_per_unit": f"R_m x B_ray + B_state = {r_m:.3f} x {b_ray:.0f} B + {b_state:.0f} B "
                                     f"= {bytes_per_mut:.0f} B/mutation (B_ray: {levels} BVH levels x 64 B + "
                                     f"4 x 48 B; k_bar = {k_bar:.2f} measured; R_m: {r_m_src})"}
    kname = ("k_step_co (coroutine chain-step kernel, BVH traversal with dynamic ray fetch)"
             if wl["scene"] == "clusters" else "k_step (chain-step megakernel)")
    roofline.update({"kernel": kname,
                     "kernel_share": res["step_ms"] / res["ms"] if res["ms"] else None})
    if wl["bound"] != "fp32" and res.get("trace_ms"):
        # wavefront step: the dominant kernel is the BVH tracer k_wf_trace; its
        # algorithmic bytes are this rank's device rays x B_ray over its summed
        # launch time (the chain-state traffic belongs to k_wf_logic)
        ach = res["rays_local"] * b_ray / (res["trace_ms"] / 1e3) / 1e9
        rays_per_launch = res["rays_local"] / max(res["trace_launches"], 1)
        wf_traffic = None
        try:   # ncu --set full of one k_wf_trace launch with a known ray count (profiles/traffic_<workload>.json)
            wf_traffic = json.load(open(tpath))["k_wf_trace"]["dram_bytes_per_ray"] * rays_per_launch
        except Exception:
            wf_traffic = None
        roofline.update({
            "achieved": ach, "frac": ach / peak, "traffic": wf_traffic,
            "work_per_unit": f"B_ray = {levels} BVH levels x 64 B + 4 x 48 B = {b_ray:.0f} B per device ray "
                             f"(SURVEY.md §8(d) per-ray term); {res['rays_local'] / max(res['trace_launches'], 1):.0f} "
                             f"rays per launch on average",
            "kernel": "k_wf_trace (wavefront BVH tracer: persistent, dynamic ray fetch, while-while rounds)",
            "kernel_share": res["trace_ms"] / res["ms"] if res["ms"] else None,
            "launches": res["trace_launches"],
            "step": {"wavefront_rounds_per_step": res["wf_rounds"] / max(args.steps, 1),
                     "k_wf_logic_share": (res["step_ms"] - res["trace_ms"]) / res["ms"] if res["ms"] else None,
                     "state_model_bytes_per_mutation": bytes_per_mut,
                     "state_model_note": "R_m x B_ray + B_state (the whole-step byte model of round 1)"}})
    if res.get("ceiling"):
        dev_rays = res["rays_dev"] / (res["ms"] / 1e3) / max(res["world"], 1)
        roofline["traversal_ceiling"] = {
            "k_trace_bench_rays_per_s": res["ceiling"], "in_step_rays_per_s_per_gpu": dev_rays,
            "frac": dev_rays / res["ceiling"],
            "in_trace_kernel_rays_per_s": (res["rays_local"] / (res["trace_ms"] / 1e3)) if res.get("trace_ms") else None,
            "note": "k_trace_bench: the fused coroutine kernel's BVH traversal loop alone on seeded incoherent "
                    "closest-hit rays, same BVH, same GPU -- a traversal-only probe of this BVH; the whole-step "
                    "ray rate (rays / step time, logic kernels included) is compared with it, and "
                    "in_trace_kernel_rays_per_s is the rate inside the wavefront's k_wf_trace launches (its "
                    "mix has camera rays and any-hit visibility rays, so it can exceed the probe)"}
    cpu = None
    if not args.no_cpu_baseline and res["world"] == 1:
        sample = args.cpu_sample or wl["cpu_sample"]
        v, kind, cores, t, chains = cpu_reference_run(wl, wl["scene_text"], sample, threads)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
               "sample": f"{sample} mutations, chains = {chains} host threads, loop-only time "
                         f"{t:.2f} s (core/driver.cpp:246,262)"}
    rel = None
    if not args.no_relmse and res["world"] == 1:
        rel = relmse_vs_reference(args)
    e2e_v, h2d, d2h, _ = run_e2e(args, wl) if res["world"] == 1 else res["e2e"]
    e2e_steps = max(args.steps, wl["e2e_steps"])
    steps = args.steps
    line = {
        "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": res["world"],
        "steps": steps, "warmup": args.warmup, "ms_per_step": res["ms"] / steps,
        "higher_is_better": True, "scaling": wl["scaling"], "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded stand-in scene, BASELINE.json config)", "config": config,
        "rays_per_s": {"device": res["rays_dev"] / (res["ms"] / 1e3),
                       "device_per_mutation": res["rays_dev"] / res["muts"],
                       "reference_equivalent": res["value"] * r_m, "r_m": r_m, "r_m_source": r_m_src},
        "acceptance": {"value": res["acceptance"], "target": 0.5,
                       "window": "mean perturbation acceptance over the timed steps, all ranks",
                       "burnin": res["burnin"]},
        "relmse": rel,
        "roofline": roofline, "cpu_baseline": cpu,
        "e2e": {"value": e2e_v, "unit": UNIT, "h2d_bytes_per_step": h2d / e2e_steps,
                "d2h_bytes_per_step": d2h / e2e_steps, "steps": e2e_steps,
                "path": ("ramlt_gpu_create_from_text + ramlt_gpu_render (b, init, K steps) + "
                         "ramlt_gpu_read_image, host buffers, wall clock") if res["world"] == 1 else
                        ("distributed.ShardedRender: per-rank create from host scene text, gathered b, "
                         "init, K steps with pooled exchange, film all-reduce, rank-0 D2H; wall clock, "
                         "max over ranks")},
        "gpu_launches": res["launches"], "clocks": res["clocks"],
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

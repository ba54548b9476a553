"""Parity of the benched path itself: the kernel behind
bench.py's c4/c5 lines is the wavefront step (k_wf_logic<float, Philox> +
k_wf_trace<float>: the coroutine StepCo advanced between BVH trace rounds;
round 1 / early round 2: the fused coroutine kernel k_step_co) with pooled
RA-quadtree lens adaptation on the 2^20 + 20 triangle clustered room.

  (i)   f64 at full scene size: the same kernel family (coroutine step, BVH,
        Philox, pooled RA-quadtree with refines) in the parity build against
        the restatement oracle's LINEAR SCAN over all 1,048,596 triangles
        (core/scene.cpp:57-102) -- flags bit-exact, a within rtol 1e-9, the
        lambda trace, tallies and partition equal.
  (ii)  f32 BVH = f32 brute force: the same coroutine kernel with the two
        intersectors on a 2,020-triangle scene -- decisions identical (both
        pick the (t, index) minimum with the same Moeller-Trumbore arithmetic;
        the BVH's padded boxes and slab slack only ever add candidates).
  (iii) f32 against f64 at scale: the benched configuration at 1024^2 --
        relMSE (error_report, core/diagnostics.cpp:11-38) of the f32 image
        within 1.5x the f64 engine's own seed-to-seed relMSE, acceptance
        within 3 standard errors.
  (iv)  acceptance against the UNMODIFIED reference on the same 2^20 scene:
        16 reference threads (one chain each, core/driver.cpp:282-297) vs the
        f32 engine, same per-chain step count, within 3 standard errors.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BIG = 1 << 20


@pytest.fixture(scope="module")
def big_scene():
    from paper_2402_08273_b200 import scenes
    return scenes.cluster_room(n_tris=BIG)   # bench.py c4/c5: 64 clusters, seed 7


def _engine(scene, **kw):
    from paper_2402_08273_b200 import Engine, RenderConfig
    return Engine(scene, RenderConfig(**kw))


FULL = dict(strategy="ra-quadtree", perturbation="lens", chains=32, mutations=32 * 8 + 7, width=1024,
            height=1024, max_vertices=13, b_samples=200, seed=11, trace_enabled=True, m_refine=32 * 3 + 5,
            m_split=4, metrics_interval=32 * 4)
K_FULL = 9


@pytest.fixture(scope="module")
def full_scene_oracle(big_scene, oracle_lib):
    """The restatement oracle's linear scan over all 1,048,596 triangles."""
    from oracle.abi import OracleConfig
    return oracle_lib.render(big_scene, OracleConfig(**FULL, rng="philox", adapt_mode="pooled"),
                             log_steps=K_FULL, cap_tallies=1 << 12, cap_trace=1 << 14, dump=True)


@pytest.mark.slow
@pytest.mark.parametrize("launch", ["coop", "per_step", "wavefront"])
def test_f64_full_scene_bvh_matches_linear_scan_oracle(launch, big_scene, full_scene_oracle, monkeypatch):
    """wavefront = the benched launch structure (k_wf_logic / k_wf_trace rounds per
    lockstep step + k_adapt_pool_accum / k_adapt_pool_apply), per_step = one fused
    k_step_co launch per lockstep step, coop = the whole span in one cooperative
    launch (small chain counts)."""
    o = full_scene_oracle
    monkeypatch.setenv("RAMLT_STEP_KERNEL", "wf" if launch == "wavefront" else "co")
    monkeypatch.setenv("RAMLT_INIT_KERNEL", "wf" if launch == "wavefront" else "co")   # wf: k_wf_logic<INIT> rounds
    if launch != "coop":
        monkeypatch.setenv("RAMLT_COOP", "0")
    eng = _engine(big_scene, **FULL, precision="f64", rng="philox", adapt_mode="pooled", accel="bvh",
                  log_steps=K_FULL, dump_partition=True)
    eng.set_b(o.stats.b)
    eng.init_chains()
    eng.run(FULL["mutations"])
    a, f = eng.decisions(K_FULL)
    assert np.array_equal(f, o.log_flags), np.argwhere(f != o.log_flags)[:3]
    np.testing.assert_allclose(a, o.log_a, rtol=1e-9, atol=1e-300)
    tr = eng.trace()
    ot = o.trace[np.lexsort((o.trace[:, 2], o.trace[:, 1], o.trace[:, 0]))]
    assert tr.shape == ot.shape and tr.shape[0] > 0
    np.testing.assert_array_equal(tr[:, :3], ot[:, :3])
    np.testing.assert_allclose(tr[:, 3:], ot[:, 3:], rtol=1e-12, atol=1e-12)
    tal = eng.tallies()
    np.testing.assert_allclose(tal[: len(o.tallies)], o.tallies[: len(tal)], rtol=1e-12, atol=1e-12)
    assert eng.partition_dump() == o.dump
    np.testing.assert_allclose(eng.image(), o.image, rtol=1e-5, atol=1e-6 * float(np.abs(o.image).max()))
    s = eng.stats()
    assert s.total_mutations == o.stats.total_mutations
    assert s.region_count == o.stats.region_count > 1
    eng.close()


@pytest.mark.parametrize("kernel", ["wf", "co"])
@pytest.mark.parametrize("strategy,rng", [("fixed", "pcg32"), ("fixed", "philox"), ("ra-quadtree", "philox")])
def test_f32_bvh_equals_f32_brute_force(strategy, rng, kernel, monkeypatch):
    """kernel = both runs' step and chain initialisation (wf: wavefront rounds, the benched
    default, traced by k_wf_trace over the BVH / k_wf_trace_brute over the linear scan; co:
    the fused coroutine kernel with its BVH / shared-memory scan)."""
    from paper_2402_08273_b200 import scenes
    monkeypatch.setenv("RAMLT_STEP_KERNEL", kernel)
    monkeypatch.setenv("RAMLT_INIT_KERNEL", kernel)
    monkeypatch.setenv("RAMLT_COOP", "0")
    scene = scenes.cluster_room(n_tris=2000, clusters=8, seed=3)
    C, K = 2048, 24
    common = dict(strategy=strategy, perturbation="lens", chains=C, mutations=C * K, width=128, height=128,
                  max_vertices=13, b_samples=4096, seed=5, precision="f32", rng=rng, log_steps=K,
                  adapt_mode="pooled", m_refine=C * 6, m_split=200)
    out = {}
    for accel in ("brute", "bvh"):
        eng = _engine(scene, **common, accel=accel)
        eng.set_b(1.0)
        eng.init_chains()
        eng.run(C * K)
        a, f = eng.decisions(K)
        s = eng.stats()
        out[accel] = (a, f, eng.image(), s.rays_closest + s.rays_visibility)
        eng.close()
    (ab, fb, ib, rb), (av, fv, iv, rv) = out["brute"], out["bvh"]
    # identical decisions and ray counts; a agrees to a few fp32 ulps (the two
    # instantiations contract FMAs in the shared mutation code differently)
    assert np.array_equal(fb, fv), np.argwhere(fb != fv)[:5]
    np.testing.assert_allclose(av, ab, rtol=4e-6, atol=0)
    assert rb == rv
    np.testing.assert_allclose(iv, ib, rtol=1e-5, atol=1e-6 * float(np.abs(ib).max()))


@pytest.mark.parametrize("rng", ["philox", "pcg32"])
@pytest.mark.parametrize("strategy", ["fixed", "ra-quadtree"])
def test_f32_wavefront_equals_fused_coroutine_kernel(strategy, rng, monkeypatch):
    """The production build's wavefront step (queues per yield point, compact bounce-loop
    state, hot / cold sectors) against the fused coroutine kernel k_step_co on the same BVH:
    the same coroutine, so identical decisions, ray counts and partition, a and the lambda
    trace to fp32 rounding.  (The f64 wavefront -- compact image and k_wf_bounce included --
    is pinned bit-exactly to the reference by test_gpu_parity.)"""
    from paper_2402_08273_b200 import scenes
    monkeypatch.setenv("RAMLT_COOP", "0")
    monkeypatch.setenv("RAMLT_INIT_KERNEL", "co")
    scene = scenes.cluster_room(n_tris=2000, clusters=8, seed=3)
    C, K = 3000, 24
    out = []
    for kernel in ("co", "wf"):
        monkeypatch.setenv("RAMLT_STEP_KERNEL", kernel)
        eng = _engine(scene, strategy=strategy, perturbation="lens", chains=C, mutations=C * K, width=128,
                      height=128, max_vertices=13, b_samples=4096, seed=11, precision="f32", rng=rng,
                      log_steps=K, adapt_mode="pooled", m_refine=C * 6, m_split=200, accel="bvh",
                      dump_partition=True)
        eng.set_b(1.0)
        eng.init_chains()
        eng.run(C * K)
        a, f = eng.decisions(K)
        s = eng.stats()
        out.append((a, f, eng.image(), eng.trace(), eng.partition_dump(), s.rays_closest + s.rays_visibility))
        eng.close()
    (a1, f1, i1, t1, d1, r1), (a2, f2, i2, t2, d2, r2) = out
    # identical decisions, ray counts and partition; a and the pooled lambda trace agree to a
    # few fp32 ulps (the kernels contract FMAs in the shared mutation code differently)
    assert np.array_equal(f1, f2), np.argwhere(f1 != f2)[:5]
    np.testing.assert_allclose(a2, a1, rtol=4e-6, atol=0)
    assert r1 == r2
    assert t1.shape == t2.shape
    np.testing.assert_array_equal(t1[:, :3], t2[:, :3])
    np.testing.assert_allclose(t2[:, 3:], t1[:, 3:], rtol=1e-6, atol=1e-9)
    assert d1 == d2
    np.testing.assert_allclose(i2, i1, rtol=1e-4, atol=1e-6 * float(np.abs(i1).max()))


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_wavefront_pipelines_equal_single_range(precision, monkeypatch):
    """RAMLT_WF_PIPES=2: the chains stepped as two wavefront pipelines on two streams
    (their k_wf_trace / k_wf_logic kernels sharing the SMs) make the decisions of the
    single pipeline -- per-chain state, order-independent pooled adaptation; with refines."""
    from paper_2402_08273_b200 import scenes
    monkeypatch.setenv("RAMLT_STEP_KERNEL", "wf")
    monkeypatch.setenv("RAMLT_COOP", "0")
    monkeypatch.setenv("RAMLT_WF_PIPES_MIN", "256")
    scene = scenes.cluster_room(n_tris=2000, clusters=8, seed=3)
    C, K = 4096 + 640, 24   # ranges of unequal size
    out = []
    for pipes in ("1", "2"):
        monkeypatch.setenv("RAMLT_WF_PIPES", pipes)
        eng = _engine(scene, strategy="ra-quadtree", perturbation="lens", chains=C, mutations=C * K, width=128,
                      height=128, max_vertices=13, b_samples=4096, seed=7, precision=precision, rng="philox",
                      log_steps=K, adapt_mode="pooled", m_refine=C * 6, m_split=200, accel="bvh",
                      dump_partition=True)
        eng.set_b(1.0)
        eng.init_chains()
        eng.run(C * K)
        a, f = eng.decisions(K)
        out.append((a, f, eng.image(), eng.trace(), eng.partition_dump(), eng.stats()))
        eng.close()
    (a1, f1, i1, t1, d1, s1), (a2, f2, i2, t2, d2, s2) = out
    assert np.array_equal(f1, f2), np.argwhere(f1 != f2)[:5]
    np.testing.assert_array_equal(a1, a2)
    np.testing.assert_array_equal(t1, t2)
    assert d1 == d2
    assert s1.region_count == s2.region_count > 1
    assert s1.rays_closest + s1.rays_visibility == s2.rays_closest + s2.rays_visibility
    # the film is a sum of atomics (fp32 staging in the f32 build): order-dependent rounding only
    np.testing.assert_allclose(i2, i1, rtol=1e-4 if precision == "f32" else 1e-9,
                               atol=1e-6 * float(np.abs(i1).max()))


def _bench_like(scene, seed, precision, chains, steps, b):
    """bench.py's c4 configuration (f32 default; f64 = parity build) at 1024^2."""
    eng = _engine(scene, strategy="ra-quadtree", perturbation="lens", chains=chains, mutations=chains * steps,
                  width=1024, height=1024, max_vertices=13, b_samples=1 << 16, seed=seed, precision=precision,
                  rng="philox", adapt_mode="pooled", log_steps=steps, metrics_interval=chains * steps)
    eng.set_b(b)   # one normalisation for every image: the films are compared
    eng.init_chains()
    eng.run(chains * steps)
    a, f = eng.decisions(steps)
    img = eng.image()
    pert = (f & 2) != 0
    per_chain = np.where(pert, a, 0.0).sum(1) / np.maximum(pert.sum(1), 1)
    s = eng.stats()
    eng.close()
    return img, s.mean_acceptance, float(per_chain.std() / np.sqrt(len(per_chain)))


@pytest.mark.slow
def test_f32_benched_config_matches_f64_at_scale(big_scene):
    from oracle.abi import np_error_report
    C, S = 1 << 18, 24
    est = _engine(big_scene, strategy="fixed", chains=1024, mutations=1024, width=1024, height=1024,
                  max_vertices=13, b_samples=1 << 16, precision="f64", rng="philox")
    b, _ = est.estimate_b()   # the scene's normalisation (images at their physical scale)
    est.close()
    ref, acc_ref, se_ref = _bench_like(big_scene, 101, "f64", C, S, b)
    f64b, acc_64, se_64 = _bench_like(big_scene, 202, "f64", C, S, b)
    f32, acc_32, se_32 = _bench_like(big_scene, 303, "f32", C, S, b)
    noise = np_error_report(f64b, ref)
    err = np_error_report(f32, ref)
    print(f"relMSE f32 vs f64 {err:.5f}  f64 seed-to-seed {noise:.5f}  ratio {err / noise:.3f}; "
          f"acceptance f32 {acc_32:.5f} f64 {acc_ref:.5f} / {acc_64:.5f} (SE {se_ref:.1e})")
    assert err <= 1.5 * noise
    assert abs(acc_32 - acc_ref) <= 3.0 * np.hypot(se_32, se_ref) + abs(acc_64 - acc_ref)


@pytest.mark.slow
def test_acceptance_matches_unmodified_reference_full_scene(big_scene, ref_lib):
    from oracle.abi import OracleConfig
    threads = min(16, os.cpu_count() or 1)
    S = 160
    cfg = OracleConfig(strategy="fixed", perturbation="lens", chains=threads, mutations=threads * S,
                       width=256, height=256, max_vertices=13, b_samples=16, seed=3,
                       metrics_interval=threads * S)
    r = ref_lib.render(big_scene, cfg, log_steps=S)
    pert = (r.log_flags & 2) != 0
    ref_chain = np.where(pert, r.log_a, 0.0).sum(1) / np.maximum(pert.sum(1), 1)
    acc_ref = r.stats.mean_acceptance
    se_ref = ref_chain.std(ddof=1) / np.sqrt(threads)
    C = 1 << 14
    eng = _engine(big_scene, strategy="fixed", perturbation="lens", chains=C, mutations=C * S, width=256,
                  height=256, max_vertices=13, b_samples=1 << 14, seed=9, precision="f32", rng="philox")
    eng.set_b(1.0)
    eng.init_chains()
    eng.run(C * S)
    acc = eng.stats().mean_acceptance
    eng.close()
    print(f"acceptance: reference {acc_ref:.4f} +- {se_ref:.4f} ({threads} threads x {S} steps), f32 engine {acc:.4f}")
    assert abs(acc - acc_ref) <= 3.0 * se_ref


def test_f32_decisions_agree_with_reference_c1():
    """SURVEY.md §8(c) P1 at C1 size: Fixed lens, 1,024 chains, K = 32, the
    reference's PCG streams; the f32 build's first K decisions against the
    restatement oracle (bit-exact with the reference, tests/test_oracle_pin.py).
    Bar: >= 99 % of chains agree on all K decisions."""
    from oracle.abi import OracleConfig, OracleLib
    from paper_2402_08273_b200 import scenes
    scene = scenes.cornell_box()
    C, K = 1024, 32
    common = dict(strategy="fixed", perturbation="lens", chains=C, mutations=C * K, width=256, height=256,
                  max_vertices=9, b_samples=4096, seed=1)
    o = OracleLib().render(scene, OracleConfig(**common), log_steps=K)
    eng = _engine(scene, **common, precision="f32", rng="pcg32", log_steps=K)
    eng.set_b(o.stats.b)
    eng.init_chains()
    eng.run(C * K)
    a, f = eng.decisions(K)
    eng.close()
    same = np.all((f & 1) == (o.log_flags & 1), axis=1)
    first = [int(np.argmax((f[c] & 1) != (o.log_flags[c] & 1))) for c in np.flatnonzero(~same)]
    print(f"f32 chains agreeing on all {K} decisions: {same.mean():.4f}; first divergent steps {first[:20]}")
    assert same.mean() >= 0.99

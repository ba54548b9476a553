"""Multi-GPU paths on one B200 (SURVEY.md §8(e) exactness test).

The box has one GPU, so two shards share cuda:0 -- the code path is the one
8 GPUs take (the exchanges are stream-ordered copies / collectives between
steps; no kernel ever waits on another shard's kernel):

  * the multi-device C-ABI handle (ramlt_gpu_create_multi, devices [0, 0]):
    peer-memory exchanges inside one process;
  * ShardedRender over two torch.distributed ranks (gloo, both on cuda:0):
    one process per GPU, the bench's N > 1 path.

Bars: Fixed -- decisions bit-identical to the single handle, film to fp64
summation order; pooled adaptive (RA-quadtree with refines at boundaries that
are not multiples of the chain count) -- decisions, lambda trace, tallies,
partition dump identical to the single handle run with the pooled rule.
"""
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cfg(**kw):
    from paper_2402_08273_b200 import RenderConfig
    c = dict(perturbation="lens", chains=301, width=40, height=40, max_vertices=12, b_samples=3000, seed=21,
             precision="f64", rng="philox", log_steps=24, adapt_mode="pooled", trace_enabled=True,
             dump_partition=True)
    c.update(kw)
    return RenderConfig(**c)


def _run(scene, cfg, b, devices=None, film_sync_steps=4096, reference=None):
    from paper_2402_08273_b200 import Engine
    eng = Engine(scene, cfg, devices=devices, film_sync_steps=film_sync_steps)
    eng.set_b(b)
    if reference is not None:
        eng.set_reference(reference)
    eng.init_chains()
    eng.run(cfg.mutations)
    a, f = eng.decisions(cfg.log_steps)
    out = dict(a=a, f=f, img=eng.image(), film=eng.film()[0], stats=eng.stats(), metrics=eng.metrics())
    if cfg.strategy != "fixed":
        out.update(trace=eng.trace(), tallies=eng.tallies(), regions=eng.regions(), dump=eng.partition_dump())
    eng.close()
    return out


def _same(x, y, adaptive):
    assert np.array_equal(x["f"], y["f"]), np.argwhere(x["f"] != y["f"])[:3]
    np.testing.assert_array_equal(x["a"], y["a"])
    np.testing.assert_allclose(x["film"], y["film"], rtol=1e-12, atol=1e-12 * float(np.abs(y["film"]).max()))
    np.testing.assert_allclose(x["img"], y["img"], rtol=1e-6, atol=1e-7 * float(np.abs(y["img"]).max()))
    sx, sy = x["stats"], y["stats"]
    assert sx.total_mutations == sy.total_mutations
    assert sx.perturbation_proposals == sy.perturbation_proposals
    assert sx.mean_acceptance == pytest.approx(sy.mean_acceptance, rel=1e-12)
    assert sx.film_luminance == pytest.approx(sy.film_luminance, rel=1e-12)
    if adaptive:
        np.testing.assert_array_equal(x["trace"], y["trace"])
        np.testing.assert_array_equal(x["tallies"], y["tallies"])
        np.testing.assert_array_equal(x["regions"][0], y["regions"][0])
        np.testing.assert_array_equal(x["regions"][1], y["regions"][1])
        assert x["dump"] == y["dump"]
        assert sx.region_count == sy.region_count


@pytest.mark.parametrize("n_dev", [2, 3])
@pytest.mark.parametrize("strategy,pert,scene_name", [("fixed", "lens", "cornell"),
                                                      ("ra-quadtree", "lens", "cornell"),
                                                      ("ra-quadtree", "multi-chain", "caustic"),
                                                      ("global", "lens", "mirror")])
def test_multi_device_handle_equals_single(n_dev, strategy, pert, scene_name):
    """ramlt_gpu_create_multi over n_dev shards (all on cuda:0) vs one handle:
    Fixed and pooled adaptive runs identical, with refine barriers and metrics
    rows at mutation counts that split a lockstep step, and the film merged
    every 3 lockstep steps."""
    from paper_2402_08273_b200 import scenes
    scene = scenes.SCENES[scene_name]()
    C = 301
    cfg = _cfg(strategy=strategy, perturbation=pert, chains=C, mutations=C * 24 + 17, m_refine=C * 5 + 50,
               m_split=40, n_top=4, n_bottom=3, metrics_interval=C * 7 + 3)
    one = _run(scene, cfg, 1.7)
    many = _run(scene, cfg, 1.7, devices=[0] * n_dev, film_sync_steps=3)
    _same(many, one, strategy != "fixed")
    # metrics rows at the same mutation counts, global interval acceptance
    m1, mn = one["metrics"], many["metrics"]
    assert mn.shape == m1.shape
    np.testing.assert_array_equal(mn[:, 1], m1[:, 1])
    np.testing.assert_allclose(mn[:, 3], m1[:, 3], rtol=1e-12)


def test_multi_device_rrmse_rows_and_errors():
    """Metrics rows of the multi-device handle carry the rRMSE of the global
    image (equal to the single handle's rows); per-shard plumbing calls are
    refused with the reference's logic_error status."""
    from paper_2402_08273_b200 import Engine, RenderConfig, scenes
    from paper_2402_08273_b200.render import LogicError
    scene = scenes.cornell_box()
    C = 64
    cfg = _cfg(strategy="fixed", chains=C, mutations=C * 20, metrics_interval=C * 5, width=24, height=24,
               trace_enabled=False, dump_partition=False)
    ref = np.random.default_rng(0).uniform(0.0, 0.2, size=(24, 24, 3)).astype(np.float32)
    one = _run(scene, cfg, 1.3, reference=ref)
    many = _run(scene, cfg, 1.3, devices=[0, 0], film_sync_steps=0, reference=ref)
    np.testing.assert_allclose(many["metrics"][:, 2], one["metrics"][:, 2], rtol=1e-9)
    assert np.all(np.isfinite(many["metrics"][:, 2]))
    eng = Engine(scene, cfg, devices=[0, 0])
    with pytest.raises(LogicError):
        eng.adapt_apply()
    with pytest.raises(LogicError):
        eng.set_stream(0)
    eng.close()
    with pytest.raises(LogicError):
        Engine(scene, RenderConfig(strategy="fixed", chains=1, mutations=1, width=8, height=8,
                                   max_vertices=9), devices=[0, 0])


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sharded_worker(rank, world, port, q, kw, b):
    import os
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2402_08273_b200 import scenes
        from paper_2402_08273_b200.distributed import ShardedRender
        torch.cuda.set_device(0)
        cfg = _cfg(**kw)
        sr = ShardedRender(scenes.cornell_box(), cfg, film_sync_steps=4)
        sr.engine.set_b(b)
        sr.init_chains()
        sr.run(cfg.mutations)
        img = sr.image()
        a, f = sr.engine.decisions(cfg.log_steps)
        out = dict(rank=rank, off=sr.plan.offset, a=a, f=f, img=img, rows=np.array(sr.rows))
        if cfg.strategy != "fixed":
            out.update(trace=sr.engine.trace(), tallies=sr.engine.tallies(), regions=sr.engine.regions(),
                       dump=sr.partition_dump())
        torch.cuda.synchronize()
        q.put(out)
        sr.engine.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("strategy", ["fixed", "ra-quadtree"])
def test_sharded_render_two_ranks_equals_single(strategy):
    """ShardedRender on two gloo ranks (both on cuda:0): the per-step pooled
    exchange, refine barriers inside a lockstep step, and the film merged
    every 4 lockstep steps reproduce the single pooled handle."""
    import torch.multiprocessing as mp
    from paper_2402_08273_b200 import scenes
    C = 257
    kw = dict(strategy=strategy, chains=C, mutations=C * 20 + 5, m_refine=C * 6 + 11, m_split=30, n_top=4,
              metrics_interval=C * 5)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q, dict(kw), 1.9)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted((q.get(timeout=600) for _ in range(2)), key=lambda o: o["rank"])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    one = _run(scenes.cornell_box(), _cfg(**kw), 1.9)
    f = np.concatenate([o["f"] for o in outs], axis=0)
    a = np.concatenate([o["a"] for o in outs], axis=0)
    assert np.array_equal(f, one["f"])
    np.testing.assert_array_equal(a, one["a"])
    for o in outs:   # every rank holds the global film after the final merge
        np.testing.assert_allclose(o["img"], one["img"], rtol=1e-6, atol=1e-7 * float(np.abs(one["img"]).max()))
        assert o["rows"].shape[0] == one["metrics"].shape[0]
        np.testing.assert_array_equal(o["rows"][:, 1], one["metrics"][:, 1])
        np.testing.assert_allclose(o["rows"][:, 3], one["metrics"][:, 3], rtol=1e-12)
        if strategy != "fixed":
            np.testing.assert_array_equal(o["trace"], one["trace"])
            np.testing.assert_array_equal(o["tallies"], one["tallies"])
            np.testing.assert_array_equal(o["regions"][0], one["regions"][0])
            assert o["dump"] == one["dump"]

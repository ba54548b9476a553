"""The N > 1 path on CPU: world_size-2 gloo process groups run the real
distributed host logic (paper_2402_08273_b200.distributed) with the CPU oracle
standing in for each rank's engine, and the results must equal the
single-process run (SURVEY.md §8(e) exactness test)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2402_08273_b200.distributed import (ShardPlan, gather_b_partials, reduce_film_host)

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.abi import OracleConfig, OracleLib, oracle_b_partials
        from paper_2402_08273_b200 import scenes
        lib = OracleLib()
        scene = scenes.cornell_box()
        C = 10
        base = dict(strategy="fixed", perturbation="lens", chains=C, mutations=C * 20 + 3,
                    width=24, height=24, max_vertices=9, b_samples=3000, seed=9, rng="philox")
        plan = ShardPlan(C, world, rank)
        # b: this rank's substreams, gathered in order, reduced like the engine
        n_sub = min(base["b_samples"], 65536)
        b0, b1 = plan.substreams(n_sub)
        part = oracle_b_partials(lib, scene, OracleConfig(**base), b0, b1)
        full = gather_b_partials(part, plan, n_sub)
        # shard of chains with global ids
        cfg = OracleConfig(**dict(base, chains=plan.count, chain_offset=plan.offset,
                                  chains_total=C, b_override=1.0))
        o = lib.render(scene, cfg, log_steps=20)
        film = reduce_film_host(o.extra["film"])
        flags = [None] * world
        dist.all_gather_object(flags, (plan.offset, o.log_flags.tolist(), o.log_a.tolist()))
        # pooled adaptation exchange arithmetic: integer SUM is partition independent
        import torch
        cnt = torch.tensor([rank + 1, 2 * rank, 7], dtype=torch.int64)
        dist.all_reduce(cnt)
        q.put((rank, full, film, flags, cnt.tolist(), o.stats.total_mutations))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(WORLD):
        r = q.get(timeout=300)
        out[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_shard_plan_partitions_chains():
    for total in (1, 7, 1024, 262144):
        for world in (1, 2, 3, 8):
            spans = [(ShardPlan(total, world, r).offset, ShardPlan(total, world, r).count)
                     for r in range(world)]
            assert spans[0][0] == 0
            assert sum(c for _, c in spans) == total
            for (o0, c0), (o1, _) in zip(spans, spans[1:]):
                assert o0 + c0 == o1


def test_b_partials_gather_equals_single_process(results):
    from oracle.abi import OracleConfig, OracleLib, oracle_b_partials
    from paper_2402_08273_b200 import scenes
    lib = OracleLib()
    base = dict(strategy="fixed", perturbation="lens", chains=10, mutations=203, width=24, height=24,
                max_vertices=9, b_samples=3000, seed=9, rng="philox")
    single = oracle_b_partials(lib, scenes.cornell_box(), OracleConfig(**base), 0, 3000)
    for r in range(WORLD):
        assert np.array_equal(results[r][1], single)     # identical on every rank, bit for bit
    o = lib.render(scenes.cornell_box(), OracleConfig(**base))
    s = single.sum(axis=0)                                # same order as the engine's reduce
    acc = 0.0
    for v in single[:, 0]:
        acc += v
    assert acc / 3000 == o.stats.b


def test_sharded_film_and_decisions_equal_single_process(results):
    from oracle.abi import OracleConfig, OracleLib
    from paper_2402_08273_b200 import scenes
    lib = OracleLib()
    base = dict(strategy="fixed", perturbation="lens", chains=10, mutations=203, width=24, height=24,
                max_vertices=9, b_samples=3000, seed=9, rng="philox", b_override=1.0)
    o = lib.render(scenes.cornell_box(), OracleConfig(**base), log_steps=20)
    for r in range(WORLD):
        np.testing.assert_allclose(results[r][2], o.extra["film"], rtol=1e-12, atol=1e-12)
    # per-chain decisions are G-invariant: global chain ids keep their streams
    shards = sorted(results[0][3])
    flags = np.concatenate([np.array(f, np.uint8) for _, f, _ in shards], axis=0)
    a = np.concatenate([np.array(x, np.float64) for _, _, x in shards], axis=0)
    assert np.array_equal(flags, o.log_flags)
    assert np.array_equal(a, o.log_a)
    assert all(results[r][5] == 203 for r in range(WORLD))   # global span bookkeeping


def test_adaptation_exchange_sum(results):
    for r in range(WORLD):
        assert results[r][4] == [1 + 2, 0 + 2, 14]

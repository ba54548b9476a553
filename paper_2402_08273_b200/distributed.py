"""Multi-GPU plumbing: chains shard across ranks (one process per GPU); NCCL
(torch.distributed) carries only the exchanges the method has:

  * b            -- per-substream partial sums gathered in substream order and
                    reduced identically on every rank (bit-identical to 1 GPU);
  * adaptation   -- pooled per-region (visit count, fixed-point acceptance sum,
                    last mutation index) SUM/SUM/MAX all-reduce per lockstep
                    step, then the same deterministic update on every rank
                    (G-invariant: integer sums do not depend on the partition);
  * framebuffer  -- fp64 film SUM all-reduce at sync points.

Chain c keeps its global id everywhere (RNG stream, decision order), so a
Fixed-strategy run is identical at any GPU count.  The same code runs on CPU
tensors with the gloo backend (tests/test_distributed.py).
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np


@dataclass(frozen=True)
class ShardPlan:
    """Contiguous chain shard of one rank: [offset, offset + count)."""
    chains_total: int
    world: int
    rank: int

    @property
    def offset(self) -> int:
        return self.rank * self.chains_total // self.world

    @property
    def count(self) -> int:
        return (self.rank + 1) * self.chains_total // self.world - self.offset

    def substreams(self, n_sub: int) -> tuple[int, int]:
        """b-estimate substreams [begin, end) computed by this rank."""
        return self.rank * n_sub // self.world, (self.rank + 1) * n_sub // self.world


def n_substreams(cfg) -> int:
    return min(cfg.b_samples, cfg.b_substreams or 65536)


def shard_config(cfg, plan: ShardPlan, device: int | None = None):
    return replace(cfg, chains=plan.count, chains_total=plan.chains_total, chain_offset=plan.offset,
                   device=cfg.device if device is None else device)


def gather_b_partials(partials: np.ndarray, plan: ShardPlan, n_sub: int, device=None) -> np.ndarray:
    """All-gather every rank's (sum, sumsq) rows into substream order."""
    import torch
    import torch.distributed as dist
    counts = [plan.__class__(plan.chains_total, plan.world, r).substreams(n_sub) for r in range(plan.world)]
    width = max(e - b for b, e in counts)
    buf = torch.zeros((width, 2), dtype=torch.float64, device=device)
    buf[: partials.shape[0]] = torch.from_numpy(partials).to(buf.device)
    out = [torch.zeros_like(buf) for _ in range(plan.world)]
    dist.all_gather(out, buf)
    rows = [o[: e - b].cpu().numpy() for o, (b, e) in zip(out, counts)]
    return np.concatenate(rows, axis=0)


def all_gather_b(engine, cfg, plan: ShardPlan):
    """Sharded estimate_b: this rank's substreams, gathered, reduced in order."""
    import torch
    n_sub = n_substreams(cfg)
    b0, b1 = plan.substreams(n_sub)
    part = engine.b_partials(b0, b1)
    dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
    full = gather_b_partials(part, plan, n_sub, device=dev)
    return engine.reduce_b(full)


class _CudaArray:
    """Zero-copy torch view of an engine-owned device buffer."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def device_tensor(ptr: int, n: int, typestr: str):
    import torch
    return torch.as_tensor(_CudaArray(ptr, n, typestr), device="cuda")


def exchange_adaptation(engine):
    """Pooled adaptation exchange after a lockstep step: SUM counts and
    fixed-point sums, MAX last index, then apply identically on every rank."""
    import torch.distributed as dist
    cnt, fx, last, n = engine.adapt_exchange()
    if n:
        tc = device_tensor(cnt, n, "<u8").view(dtype=__import__("torch").int64)
        tf = device_tensor(fx, n, "<u8").view(dtype=__import__("torch").int64)
        tl = device_tensor(last, n, "<u8").view(dtype=__import__("torch").int64)
        dist.all_reduce(tc, op=dist.ReduceOp.SUM)
        dist.all_reduce(tf, op=dist.ReduceOp.SUM)
        dist.all_reduce(tl, op=dist.ReduceOp.MAX)
    engine.adapt_apply()


def sync_refine(engine):
    """Deferred quadtree refine of a sharded run: SUM the
    per-region visit counts, refine identically on every rank, and keep the
    carried-over counts on rank 0 only."""
    import torch
    import torch.distributed as dist
    if not engine.refine_pending():
        return False
    ptr, n = engine.visits_device()
    if n:
        v = device_tensor(ptr, n, "<u8").view(dtype=torch.int64)
        dist.all_reduce(v, op=dist.ReduceOp.SUM)
    engine.refine(keep_counts=dist.get_rank() == 0)
    return True


def sharded_sync(engine):
    """Everything a sharded run exchanges after a lockstep step."""
    exchange_adaptation(engine)
    sync_refine(engine)


def reduce_film(engine):
    """SUM all-reduce of the fp64 film in place on every rank (NCCL)."""
    import torch.distributed as dist
    ptr, n = engine.film_device()
    t = device_tensor(ptr, n, "<f8")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t


def reduce_film_host(film: np.ndarray, device=None) -> np.ndarray:
    """SUM all-reduce of a host film (gloo / CPU path)."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(film, np.float64)).to(device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.cpu().numpy()


class ShardedRender:
    """run_render over torch.distributed ranks: one engine per rank/GPU."""

    def __init__(self, scene, cfg, exchange_every: int = 1):
        import torch
        import torch.distributed as dist
        from .render import Engine
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()
        self.plan = ShardPlan(cfg.chains, self.world, self.rank)
        local = torch.cuda.current_device()
        self.cfg = cfg
        self.engine = Engine(scene, shard_config(cfg, self.plan, local))
        self.engine.set_stream(torch.cuda.current_stream().cuda_stream)
        self.adaptive = cfg.strategy != "fixed"
        self.exchange_every = exchange_every
        if self.adaptive and self.world > 1:
            self.engine.set_exchange_interval(exchange_every)

    def estimate_b(self):
        return all_gather_b(self.engine, self.cfg, self.plan)

    def run(self, mutations: int):
        C = self.cfg.chains
        if not self.adaptive or self.world == 1:
            self.engine.run(mutations)
            return
        step = C * self.exchange_every
        done = 0
        while done < mutations:
            m = min(step, mutations - done)
            self.engine.run(m)
            sharded_sync(self.engine)
            done += m

    def render(self):
        self.estimate_b()
        self.engine.init_chains()
        self.run(self.cfg.mutations)
        return reduce_film(self.engine)


class ShardedMix:
    """The analytic-target harness (configs[1]) over torch.distributed ranks:
    chains shard by global id (their Philox streams do not depend on the
    partition); adaptive strategies advance one lockstep step at a time and
    SUM/SUM/MAX-all-reduce the pooled (count, fixed-point sum, last index)
    per region before every rank applies the identical update -- the same
    exchange as ShardedRender, so lambda trajectories equal the single-GPU
    pooled run bit for bit."""

    def __init__(self, target, cfg):
        import torch
        import torch.distributed as dist
        from .mix import MixEngine
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()
        self.plan = ShardPlan(cfg.chains, self.world, self.rank)
        local = torch.cuda.current_device()
        self.cfg = replace(cfg, chains=self.plan.count, chains_total=cfg.chains, chain_offset=self.plan.offset,
                           device=local, adapt_mode="pooled" if cfg.strategy != "fixed" else cfg.adapt_mode)
        self.engine = MixEngine(target, self.cfg)
        self.engine.set_stream(torch.cuda.current_stream().cuda_stream)
        self.adaptive = cfg.strategy != "fixed"
        if self.adaptive and self.world > 1:
            self.engine.set_external_adaptation(True)

    def init_chains(self):
        self.engine.init_chains()

    def run(self, steps: int):
        if not self.adaptive or self.world == 1:
            self.engine.run(steps)
            return
        for _ in range(steps):
            self.engine.run(1)
            exchange_adaptation(self.engine)

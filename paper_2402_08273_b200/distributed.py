"""Multi-GPU plumbing: chains shard across ranks (one process per GPU); NCCL
(torch.distributed) carries only the exchanges the method has:

  * b            -- per-substream partial sums gathered in substream order and
                    reduced identically on every rank (bit-identical to 1 GPU);
  * adaptation   -- pooled per-region (visit count, fixed-point acceptance sum,
                    last mutation index) SUM/SUM/MAX all-reduce per lockstep
                    step, then the same deterministic update on every rank
                    (G-invariant: integer sums do not depend on the partition);
  * quadtree     -- per-region visit counts SUM-reduced at every m_refine
                    barrier, then the same deterministic refine on every rank;
  * framebuffer  -- delta SUM all-reduce of the fp64 film every 2^12 lockstep
                    steps (configs[4]), at metrics rows and at the end.

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


def _u64(engine_ptr_n):
    import torch
    ptr, n = engine_ptr_n
    return device_tensor(ptr, n, "<u8").view(dtype=torch.int64) if n else None


def adapt_tensors(engine):
    """Zero-copy int64 views of the engine's pooled exchange buffers (count,
    fixed-point sum, last index); engines may provide ``adapt_tensors`` themselves
    (the CPU host-logic tests pass CPU tensors)."""
    if hasattr(engine, "adapt_tensors"):
        return engine.adapt_tensors()
    cnt, fx, last, n = engine.adapt_exchange()
    if not n:
        return None
    return _u64((cnt, n)), _u64((fx, n)), _u64((last, n))


def visits_tensor(engine):
    if hasattr(engine, "visits_tensor"):
        return engine.visits_tensor()
    return _u64(engine.visits_device())


def film_tensor(engine):
    if hasattr(engine, "film_tensor"):
        return engine.film_tensor()
    ptr, n = engine.film_device()
    return device_tensor(ptr, n, "<f8")


def exchange_adaptation(engine):
    """Pooled adaptation exchange after a lockstep step: SUM counts and
    fixed-point sums, MAX last index, then apply identically on every rank."""
    import torch.distributed as dist
    t = adapt_tensors(engine)
    if t is not None:
        tc, tf, tl = t
        dist.all_reduce(tc, op=dist.ReduceOp.SUM)
        dist.all_reduce(tf, op=dist.ReduceOp.SUM)
        dist.all_reduce(tl, op=dist.ReduceOp.MAX)
    engine.adapt_apply()


def sync_refine(engine):
    """Deferred quadtree refine of a sharded run: SUM the
    per-region visit counts, refine identically on every rank, and keep the
    carried-over counts on rank 0 only."""
    import torch.distributed as dist
    if not engine.refine_pending():
        return False
    v = visits_tensor(engine)
    if v is not None:
        dist.all_reduce(v, op=dist.ReduceOp.SUM)
    engine.refine(keep_counts=dist.get_rank() == 0)
    return True


def sharded_sync(engine):
    """Everything a sharded run exchanges after a lockstep step."""
    exchange_adaptation(engine)
    sync_refine(engine)


def reduce_film_host(film: np.ndarray, device=None) -> np.ndarray:
    """SUM all-reduce of a host film (gloo / CPU path)."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(film, np.float64)).to(device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.cpu().numpy()


def sync_film(engine, synced):
    """Delta SUM all-reduce of the fp64 film (core/film.cpp:22-27 merge, done
    periodically): every rank's film becomes the global film, each rank's
    contribution counted once.  ``synced`` is the global film of the previous
    sync (zeros at first; updated in place)."""
    import torch.distributed as dist
    t = film_tensor(engine)
    delta = t - synced
    dist.all_reduce(delta, op=dist.ReduceOp.SUM)
    synced.add_(delta)
    t.copy_(synced)
    return t


class ShardedRender:
    """run_render over torch.distributed ranks: one engine per rank/GPU.

    Chains shard by global id (ShardPlan).  Runs are chunked so that every
    exchange happens at the same global mutation count on every rank:
      * adaptive strategies: the pooled adaptation exchange every
        ``exchange_every`` lockstep steps (1 = G-invariant, identical to one GPU);
      * RA-quadtree: runs end exactly at every m_refine barrier, where the
        visits are SUM-reduced and every rank refines identically
        (core/partition.cpp:68-100, core/driver.cpp:300-304);
      * the film every ``film_sync_steps`` lockstep steps (configs[4]: 2^12,
        0 = only at metrics rows and the end) and at metrics rows, so the
        image, the luminance and the rRMSE are global on every rank;
      * b once (substream partials gathered in order).
    """

    def __init__(self, scene, cfg, exchange_every: int = 1, film_sync_steps: int = 4096, engine=None):
        import time
        import torch
        import torch.distributed as dist
        from .render import Engine
        init = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size() if init else 1
        self.rank = dist.get_rank() if init else 0
        self.plan = ShardPlan(cfg.chains, self.world, self.rank)
        self.cfg = cfg
        if engine is not None:      # host-logic tests: an engine stand-in on CPU tensors
            self.engine, self.device = engine, "cpu"
        else:
            local = torch.cuda.current_device()
            self.engine = Engine(scene, shard_config(cfg, self.plan, local))
            self.engine.set_stream(torch.cuda.current_stream().cuda_stream)
            self.device = "cuda"
        self.adaptive = cfg.strategy != "fixed"
        self.quadtree = cfg.strategy == "ra-quadtree"
        self.exchange_every = max(1, int(exchange_every))
        self.film_sync_steps = int(film_sync_steps)
        self.done = 0           # global mutations
        self.steps = 0          # lockstep steps (film merge cadence)
        self.next_metrics = cfg.metrics_interval
        self._last_row = -1
        self.rows = []          # MetricsRow (time, mutations, rrmse, interval acceptance), global
        self._synced = None
        self._film_dirty = False
        self._has_ref = False
        self._acc_last = (0.0, 0.0)
        self._t0 = None
        self._time = time.perf_counter
        if self.adaptive and self.world > 1:
            self.engine.set_exchange_interval(self.exchange_every)

    def set_reference(self, image):
        self.engine.set_reference(image)
        self._has_ref = True

    def estimate_b(self):
        if self.world == 1:
            return self.engine.estimate_b()
        return all_gather_b(self.engine, self.cfg, self.plan)

    def init_chains(self):
        self.engine.init_chains()

    def run(self, mutations: int):
        """Advance the render by ``mutations`` global mutations.  One rank:
        the engine's own span loop (exact).  Several ranks: whole lockstep steps
        of the canonical span loop (Engine.run_steps: the spans a single GPU
        uses, so every chain's decisions equal the single-GPU run), with the
        exchanges between steps; a target that is not a span boundary may be
        passed by less than one lockstep step."""
        if self._t0 is None:
            self._t0 = self._time()
        C = self.cfg.chains
        target = self.done + mutations
        if self.world == 1:
            while self.done < target:
                end = min(target, self.next_metrics)
                self.engine.run(end - self.done)
                self.done = end
                self._film_dirty = True
                if self.done == self.next_metrics or self.done == self.cfg.mutations:
                    self._push_row()
                    self.next_metrics = self.done + self.cfg.metrics_interval
            return
        while self.done < target:
            n = self.exchange_every if self.adaptive else max(1, (target - self.done) // C)
            if self.film_sync_steps:
                n = min(n, self.film_sync_steps - self.steps % self.film_sync_steps)
            done, ex = self.engine.run_steps(n)
            self.done = done
            self.steps += ex
            if ex:
                self._film_dirty = True
                if self.adaptive:
                    exchange_adaptation(self.engine)
            refined = self.quadtree and sync_refine(self.engine)
            if self.film_sync_steps and ex and self.steps % self.film_sync_steps == 0:
                self.sync_film()
            if self.done == self.next_metrics or (self.done == self.cfg.mutations and self._last_row != self.done):
                self._push_row()
                self.next_metrics = self.done + self.cfg.metrics_interval
            if not ex and not refined:
                raise RuntimeError("sharded run made no progress")

    def sync_film(self):
        import torch
        if self.world == 1:
            self._film_dirty = False
            return
        if self._synced is None:
            self._synced = torch.zeros_like(film_tensor(self.engine))
        sync_film(self.engine, self._synced)
        self._film_dirty = False

    def global_acceptance(self):
        """(accepted sum, perturbation proposals) over all ranks so far."""
        import torch
        import torch.distributed as dist
        s = self.engine.stats()
        t = torch.tensor([s.mean_acceptance * s.perturbation_proposals, float(s.perturbation_proposals)],
                         dtype=torch.float64, device=self.device)
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t[0]), float(t[1])

    def _push_row(self):
        if self._film_dirty:
            self.sync_film()
        a, n = self.global_acceptance()
        a0, n0 = self._acc_last
        self._acc_last = (a, n)
        rr = self.engine.rrmse(self.done) if self._has_ref else float("nan")
        self.rows.append((self._time() - self._t0, self.done, rr, (a - a0) / (n - n0) if n > n0 else 0.0))
        self._last_row = self.done

    def partition_dump(self) -> str:
        """PartitionIndex::dump with the leaf visit counts summed over ranks."""
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return self.engine.partition_dump()
        v = visits_tensor(self.engine).clone()
        dist.all_reduce(v, op=dist.ReduceOp.SUM)
        return self.engine.partition_dump(visits=v.cpu().numpy().astype(np.uint64))

    def image(self):
        if self._film_dirty:
            self.sync_film()
        return self.engine.image()

    def render(self):
        self.estimate_b()
        self.engine.init_chains()
        self.run(self.cfg.mutations - self.done)
        self.sync_film()
        return film_tensor(self.engine)


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

"""ShardedRender's host orchestration on CPU (gloo, world_size 2), with a
stand-in engine that has the real engine's contract:

  * run_steps(n): lockstep steps of the CANONICAL span loop (spans end at the
    configured total, every m_refine and every metrics_interval mutations;
    chain c takes a step of span [s, e) iff j < (e-s)//C or c < (e-s)%C --
    core/driver.cpp:283-291), stopping at a span end; in exchange mode the
    step's pooled visits are only accumulated;
  * adapt_apply(): the pooled update from the (all-reduced) accumulators;
  * refine_pending()/refine(keep): deferred refine at m_refine barriers.

Decisions depend on the shared per-region state, so any wrongly placed
exchange, a missed refine barrier, a span split at the wrong place or a
double-counted film merge changes the result.  The 2-rank run must equal the
single-rank run exactly (the GPU engine's version of this test is
tests/test_gpu_multi.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class FakeCfg:
    def __init__(self, **kw):
        self.strategy = kw.get("strategy", "ra-quadtree")
        self.chains = kw["chains"]
        self.mutations = kw["mutations"]
        self.m_refine = kw["m_refine"]
        self.metrics_interval = kw["metrics_interval"]
        self.b_samples = 16
        self.b_substreams = 0


class Stats:
    def __init__(self, acc, n):
        self.mean_acceptance = acc / n if n else 0.0
        self.perturbation_proposals = n


class FakeEngine:
    PIX = 97

    def __init__(self, cfg, offset, count, exchange):
        self.cfg, self.off, self.cnt = cfg, offset, count
        self.C = cfg.chains
        self.exchange = exchange
        self.lam = [0.0] * 4                      # regions (grow at refines)
        self.x = torch.zeros((3, 4), dtype=torch.int64)
        self.visits = torch.zeros(4, dtype=torch.int64)
        self.film = torch.zeros(self.PIX, dtype=torch.float64)
        self.steps = np.zeros(count, np.int64)
        self.log = [[] for _ in range(count)]
        self.acc = 0.0
        self.nprop = 0
        self.done = 0
        self.next_refine = cfg.m_refine
        self.next_metrics = cfg.metrics_interval
        self.span = None
        self.pending = False

    # ---- the canonical span loop ----
    def _open(self):
        end = min(self.cfg.mutations if self.done < self.cfg.mutations else 1 << 62, self.next_refine,
                  self.next_metrics)
        span = end - self.done
        per, rem = divmod(span, self.C)
        self.span = [self.done, end, per, rem, per + (1 if rem else 0), 0]

    def _step(self, j):
        s, e, per, rem, _, _ = self.span
        for c in range(self.cnt):
            gc = self.off + c
            if not (j < per or (j == per and gc < rem)):
                continue
            idx = s + j * self.C + gc
            k = int(self.steps[c])
            r = (gc * 7 + k * 3) % len(self.lam)
            a = 0.5 + 0.5 * np.tanh(self.lam[r] + 0.1 * ((gc * 13 + k * 5) % 11 - 5))
            u = ((gc * 2654435761 + k * 40503) % 1000) / 1000.0
            self.log[c].append(int(u < a))
            self.steps[c] += 1
            self.acc += a
            self.nprop += 1
            self.x[0, r] += 1
            self.x[1, r] += int(a * (1 << 24))
            self.x[2, r] = max(int(self.x[2, r]), idx)
            self.visits[r] += 1
            self.film[(gc + k) % self.PIX] += a
        if not self.exchange:
            self.adapt_apply()

    def _boundary(self):
        if self.done == self.next_refine:
            if self.exchange:
                self.pending = True
            else:
                self._refine(True)
            self.next_refine += self.cfg.m_refine
        if self.done == self.next_metrics or self.done == self.cfg.mutations:
            self.next_metrics = self.done + self.cfg.metrics_interval

    def run_steps(self, n):
        if self.span is None and self.pending:
            return self.done, 0
        if self.span is None:
            self._open()
        sp = self.span
        j1 = min(sp[4], sp[5] + n)
        for j in range(sp[5], j1):
            self._step(j)
        ex = j1 - sp[5]
        sp[5] = j1
        if j1 == sp[4]:
            self.done = sp[1]
            self.span = None
            self._boundary()
            return self.done, ex
        return sp[0] + (j1 * self.C if j1 <= sp[2] else sp[2] * self.C + sp[3]), ex

    def run(self, m):
        target = self.done + m
        while self.done < target:
            if self.span is None:
                # run(): spans additionally end at the caller's target
                end = min(target, self.next_refine, self.next_metrics)
                per, rem = divmod(end - self.done, self.C)
                self.span = [self.done, end, per, rem, per + (1 if rem else 0), 0]
            self.run_steps(1 << 30)

    # ---- adaptation / refine ----
    def adapt_tensors(self):
        return self.x[0], self.x[1], self.x[2]

    def adapt_apply(self):
        for r in range(len(self.lam)):
            c = int(self.x[0, r])
            if c:
                ah = int(self.x[1, r]) / (1 << 24) / c
                self.lam[r] += 0.25 if ah < 0.5 else -0.25
        self.x.zero_()

    def refine_pending(self):
        return self.pending

    def visits_tensor(self):
        return self.visits

    def refine(self, keep_counts):
        self.pending = False
        self._refine(keep_counts)

    def _refine(self, keep):
        split = [r for r in range(len(self.lam)) if int(self.visits[r]) >= 40]
        for r in split:
            self.lam.append(self.lam[r] - 0.125)
        n = len(self.lam)
        v = torch.zeros(n, dtype=torch.int64)
        if keep:
            v[: self.visits.numel()] = self.visits
            v[split] = 0
        self.visits = v
        self.x = torch.zeros((3, n), dtype=torch.int64)

    # ---- outputs ----
    def film_tensor(self):
        return self.film

    def stats(self):
        return Stats(self.acc, self.nprop)

    def set_exchange_interval(self, s):
        self.exchange = s > 0


KW = dict(chains=23, mutations=23 * 30 + 9, m_refine=23 * 4 + 5, metrics_interval=23 * 7 + 2)


def _run(world, rank, film_sync):
    from paper_2402_08273_b200.distributed import ShardPlan, ShardedRender
    cfg = FakeCfg(**KW)
    plan = ShardPlan(cfg.chains, world, rank)
    eng = FakeEngine(cfg, plan.offset, plan.count, exchange=False)
    sr = ShardedRender(None, cfg, film_sync_steps=film_sync, engine=eng)
    sr.run(cfg.mutations)
    if sr._film_dirty:
        sr.sync_film()
    v = eng.visits.clone()
    if world > 1:
        dist.all_reduce(v)
    return dict(log=eng.log, lam=list(eng.lam), film=eng.film.clone(), visits=v, rows=list(sr.rows),
                steps=eng.steps.copy(), done=sr.done)


def _worker(rank, world, port, q, film_sync):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _run(world, rank, film_sync)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("film_sync", [0, 3])
def test_sharded_render_host_logic_equals_single_rank(film_sync):
    single = _run(1, 0, film_sync)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, film_sync)) for r in range(2)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    logs = outs[0]["log"] + outs[1]["log"]
    assert logs == single["log"]
    assert np.array_equal(np.concatenate([outs[0]["steps"], outs[1]["steps"]]), single["steps"])
    assert len(single["lam"]) > 4                      # refines happened
    for r in (0, 1):
        o = outs[r]
        assert o["done"] == single["done"] == KW["mutations"]
        assert o["lam"] == single["lam"]               # identical adaptation + refines on every rank
        torch.testing.assert_close(o["film"], single["film"], rtol=1e-12, atol=1e-12)   # merged exactly once
        assert torch.equal(o["visits"], single["visits"])
        assert [row[1] for row in o["rows"]] == [row[1] for row in single["rows"]]
        np.testing.assert_allclose([row[3] for row in o["rows"]], [row[3] for row in single["rows"]], rtol=1e-12)

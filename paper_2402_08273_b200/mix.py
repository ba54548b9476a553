"""Analytic-target adaptive MCMC on the B200 engine (BASELINE.json configs[1];
C-ABI include/ramlt_mix.h).

The reference's chain loop (``run_chain_span``, core/driver.cpp:113-171) with
the light path replaced by a point of [0,1]^D, the path contribution by a
Gaussian-mixture density and the perturbation by an isotropic Gaussian random
walk of scale ``sigma_for(region)`` (core/adaptation.cpp:44-50).  Controller,
accept rule, normal quantile and RNG streams are the reference's; the target
and proposal are harness code (pinned at the controller /
accept boundary).

    tgt = MixTarget.config2(seed=0)                 # 4 anisotropic Gaussians in [0,1]^8
    eng = MixEngine(tgt, MixConfig(chains=65536))
    eng.init_chains(); eng.run(4096)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, fields

import numpy as np

from . import _capi
from .render import ADAPT_MODES, PRECISIONS, RNGS, _raise

MIX_STRATEGIES = {"fixed": 0, "global": 1, "ra-grid": 2}


@dataclass
class MixTarget:
    """pi(x) = sum_k w_k N(x; mu_k, Sigma_k) on [0,1]^D, zero outside."""
    weights: np.ndarray       # (K,)
    means: np.ndarray         # (K, D)
    covariances: np.ndarray   # (K, D, D), symmetric positive definite

    @property
    def dim(self) -> int:
        return int(self.means.shape[1])

    @property
    def n_comp(self) -> int:
        return int(self.means.shape[0])

    @staticmethod
    def config2(seed: int = 0, dim: int = 8, n_comp: int = 4, eig_log10=(-4.0, -1.0),
                mean_range=(0.2, 0.8)) -> "MixTarget":
        """BASELINE.json configs[1]: means U[0.2, 0.8]^8, covariance eigenvalues
        log-uniform in [1e-4, 1e-1] with Haar-random eigenvectors, weights
        ~ Dirichlet(1).  Seeded (numpy PCG64)."""
        rng = np.random.Generator(np.random.PCG64(seed))
        w = rng.dirichlet(np.ones(n_comp))
        mu = rng.uniform(mean_range[0], mean_range[1], size=(n_comp, dim))
        cov = np.empty((n_comp, dim, dim))
        for k in range(n_comp):
            q, r = np.linalg.qr(rng.standard_normal((dim, dim)))
            q = q * np.sign(np.diag(r))          # Haar measure
            lam = 10.0 ** rng.uniform(eig_log10[0], eig_log10[1], size=dim)
            s = (q * lam) @ q.T
            cov[k] = 0.5 * (s + s.T)             # exactly symmetric
        return MixTarget(w, mu, cov)

    def log_density(self, x: np.ndarray) -> np.ndarray:
        """Reference numpy evaluation (tests): log pi at points (n, D)."""
        x = np.atleast_2d(np.asarray(x, np.float64))
        out = np.empty((x.shape[0], self.n_comp))
        for k in range(self.n_comp):
            L = np.linalg.cholesky(self.covariances[k])
            z = np.linalg.solve(L, (x - self.means[k]).T)
            out[:, k] = (np.log(self.weights[k]) - np.log(np.diag(L)).sum()
                         - 0.5 * self.dim * np.log(2 * np.pi) - 0.5 * (z * z).sum(axis=0))
        m = out.max(axis=1)
        lp = m + np.log(np.exp(out - m[:, None]).sum(axis=1))
        inside = np.all((x >= 0) & (x <= 1), axis=1)
        return np.where(inside, lp, -np.inf)

    def to_c(self):
        w = np.ascontiguousarray(self.weights, np.float64)
        mu = np.ascontiguousarray(self.means, np.float64)
        cov = np.ascontiguousarray(self.covariances, np.float64)
        t = _capi.ramlt_mix_target()
        t.dim, t.n_comp = self.dim, self.n_comp
        dp = C.POINTER(C.c_double)
        t.weights = w.ctypes.data_as(dp)
        t.means = mu.ctypes.data_as(dp)
        t.covariances = cov.ctypes.data_as(dp)
        return t, (w, mu, cov)   # keep the arrays alive with the struct


@dataclass
class MixConfig:
    """AdaptationConfig (core/adaptation.hpp:14-22) + the B200 engine knobs."""
    strategy: str = "global"       # "fixed" | "global" | "ra-grid"
    grid_n: int = 4
    chains: int = 1
    batch_size: int = 10
    gamma_max: float = 1.0
    gamma_scale: float = 5.0
    target_acceptance: float = 0.5
    lambda_init: float = 1.0
    lambda_min: float = -30.0
    seed: int = 1
    precision: str = "f32"
    rng: str = "philox"
    adapt_mode: str = "auto"
    device: int = -1
    chains_total: int = 0
    chain_offset: int = 0
    log_steps: int = 0
    trace_enabled: bool = False
    trace_capacity: int = 0
    profile_kernels: bool = False
    cooperative: bool = True
    series_steps: int = 0         # record a scalar per chain for autocorrelation_time
    series_dim: int = -1          # -1: log pi(x), d: coordinate x_d

    def to_c(self) -> _capi.ramlt_mix_desc:
        d = _capi.ramlt_mix_desc()
        _capi.load().ramlt_mix_default_desc(C.byref(d))
        for f in fields(self):
            v = getattr(self, f.name)
            if f.name == "strategy":
                v = MIX_STRATEGIES[v]
            elif f.name == "precision":
                v = PRECISIONS[v]
            elif f.name == "rng":
                v = RNGS[v]
            elif f.name == "adapt_mode":
                v = ADAPT_MODES[v]
            elif isinstance(v, bool):
                v = int(v)
            setattr(d, f.name, v)
        return d


class MixEngine:
    """One analytic-target engine handle (one GPU, one chain shard)."""

    def __init__(self, target: MixTarget, cfg: MixConfig):
        self.lib = _capi.load()
        self.cfg = cfg
        self.target = target
        self._t, self._keep = target.to_c()
        self._d = cfg.to_c()
        h = C.c_void_p()
        rc = self.lib.ramlt_mix_create(C.byref(self._t), C.byref(self._d), C.byref(h))
        if rc:
            _raise(rc, self.lib.ramlt_mix_last_create_error().decode())
        self.h = h

    def _check(self, rc):
        if rc:
            _raise(rc, self.lib.ramlt_mix_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self.lib.ramlt_mix_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def set_stream(self, stream_ptr: int):
        self._check(self.lib.ramlt_mix_set_stream(self.h, C.c_void_p(stream_ptr)))

    def init_chains(self):
        self._check(self.lib.ramlt_mix_init_chains(self.h))

    def run(self, steps: int):
        self._check(self.lib.ramlt_mix_run(self.h, steps))

    def synchronize(self):
        self._check(self.lib.ramlt_mix_synchronize(self.h))

    def stats(self) -> _capi.ramlt_mix_stats:
        s = _capi.ramlt_mix_stats()
        self._check(self.lib.ramlt_mix_read_stats(self.h, C.byref(s)))
        return s

    def state(self):
        x = np.zeros((self.cfg.chains, self.target.dim), np.float64)
        lp = np.zeros(self.cfg.chains, np.float64)
        dp = C.POINTER(C.c_double)
        self._check(self.lib.ramlt_mix_read_state(self.h, x.ctypes.data_as(dp), lp.ctypes.data_as(dp)))
        return x, lp

    def chain_tallies(self):
        a = np.zeros(self.cfg.chains, np.float64)
        n = np.zeros(self.cfg.chains, np.uint64)
        self._check(self.lib.ramlt_mix_read_chain_tallies(
            self.h, a.ctypes.data_as(C.POINTER(C.c_double)), n.ctypes.data_as(C.POINTER(C.c_uint64))))
        return a, n

    def regions(self):
        """(lambda, n, accept_sum, visits) per region."""
        cnt = C.c_uint64()
        self._check(self.lib.ramlt_mix_read_regions(self.h, None, None, None, None, 0, C.byref(cnt)))
        m = cnt.value
        lam, acc = np.zeros(m), np.zeros(m)
        n, vis = np.zeros(m, np.uint64), np.zeros(m, np.uint64)
        dp, up = C.POINTER(C.c_double), C.POINTER(C.c_uint64)
        self._check(self.lib.ramlt_mix_read_regions(
            self.h, lam.ctypes.data_as(dp), n.ctypes.data_as(up), acc.ctypes.data_as(dp),
            vis.ctypes.data_as(up), m, C.byref(cnt)))
        return lam, n, acc, vis

    def trace(self) -> np.ndarray:
        n = C.c_uint64()
        self._check(self.lib.ramlt_mix_read_trace(self.h, None, 0, C.byref(n)))
        rows = (_capi.ramlt_trace_row * max(n.value, 1))()
        self._check(self.lib.ramlt_mix_read_trace(self.h, rows, n.value, C.byref(n)))
        return np.array([[r.mutation_index, r.region, r.n, r.lambda_, r.alpha_hat]
                         for r in rows[: n.value]], np.float64).reshape(-1, 5)

    def decisions(self, K: int):
        a = np.zeros((self.cfg.chains, K), np.float64)
        f = np.zeros((self.cfg.chains, K), np.uint8)
        self._check(self.lib.ramlt_mix_read_decisions(
            self.h, K, a.ctypes.data_as(C.POINTER(C.c_double)), f.ctypes.data_as(C.POINTER(C.c_uint8))))
        return a, f

    def series(self) -> np.ndarray:
        out = np.zeros((self.cfg.chains, self.cfg.series_steps), np.float64)
        self._check(self.lib.ramlt_mix_read_series(self.h, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def autocorrelation(self, first: int = 0, count: int | None = None):
        """autocorrelation_time (core/diagnostics.cpp:87-127) of the recorded
        series of chains [first, first + count): (tau, n_eff, sigma2, status)."""
        count = self.cfg.chains - first if count is None else count
        tau, neff, s2 = np.zeros(count), np.zeros(count), np.zeros(count)
        st = np.zeros(count, np.int32)
        dp = C.POINTER(C.c_double)
        self._check(self.lib.ramlt_mix_autocorrelation(self.h, first, count, tau.ctypes.data_as(dp),
                                                       neff.ctypes.data_as(dp), s2.ctypes.data_as(dp),
                                                       st.ctypes.data_as(C.POINTER(C.c_int32))))
        return tau, neff, s2, st

    # --- sharded pooled adaptation ---------------------------------------------------
    def set_external_adaptation(self, on: bool):
        self._check(self.lib.ramlt_mix_set_external_adaptation(self.h, int(on)))

    def adapt_exchange(self):
        c, fx, last = C.POINTER(C.c_uint64)(), C.POINTER(C.c_uint64)(), C.POINTER(C.c_uint64)()
        n = C.c_uint64()
        self._check(self.lib.ramlt_mix_adapt_exchange(self.h, C.byref(c), C.byref(fx), C.byref(last),
                                                      C.byref(n)))
        cv = lambda p: C.cast(p, C.c_void_p).value  # noqa: E731
        return cv(c), cv(fx), cv(last), n.value

    def adapt_apply(self):
        self._check(self.lib.ramlt_mix_adapt_apply(self.h))


def run_mix(target: MixTarget, cfg: MixConfig, steps: int) -> dict:
    """Init + ``steps`` lockstep steps; returns the summary the tests compare."""
    eng = MixEngine(target, cfg)
    try:
        eng.init_chains()
        eng.run(steps)
        s = eng.stats()
        x, lp = eng.state()
        lam, n, acc, vis = eng.regions()
        return dict(x=x, log_pi=lp, lambda_=lam, n=n, tally_accept=acc, tally_visits=vis,
                    mean_acceptance=s.mean_acceptance, accepted=s.accepted, trace=eng.trace())
    finally:
        eng.close()

"""Host API mirroring the reference renderer (core/driver.hpp:19-91) over the
B200 engine's C-ABI.

    result = run_render(scene_text, RenderConfig(...))     # driver.hpp:80

``RenderConfig`` / ``RenderResult`` carry the reference's fields and names;
errors surface as the reference's exception types (``RuntimeError`` for
"black-scene" and scene-parse errors, ``ValueError`` for std::invalid_argument,
``AssertionError``-free ``LogicError`` for RAMLT_CHECK failures).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, fields
from typing import Optional

import numpy as np

from . import _capi

STRATEGIES = {"fixed": 0, "global": 1, "ra-grid": 2, "ra-quadtree": 3}
PERTURBATIONS = {"lens": 0, "multi-chain": 1}
PRECISIONS = {"f32": 0, "f64": 1}
RNGS = {"pcg32": 0, "philox": 1}
ADAPT_MODES = {"auto": -1, "literal": 0, "pooled": 1}
ACCELS = {"auto": 0, "brute": 1, "bvh": 2}


class LogicError(RuntimeError):
    """std::logic_error (RAMLT_CHECK, core/check.hpp:8-19)."""


class CudaError(RuntimeError):
    """A CUDA / driver failure inside the engine."""


def _raise(code: int, msg: str):
    if code == 1:
        raise RuntimeError(msg)
    if code == 2:
        raise LogicError(msg)
    if code == 3:
        raise ValueError(msg)
    if code == 5:
        raise CudaError(msg)
    raise RuntimeError(msg)


@dataclass
class RenderConfig:
    """ramlt::RenderConfig (core/driver.hpp:19-39) + AdaptationConfig
    (core/adaptation.hpp:14-22), then the B200 engine knobs."""
    strategy: str = "ra-quadtree"
    perturbation: str = "lens"
    mutations: int = 1_000_000
    time_budget_s: float = 0.0
    chains: int = 1
    batch_size: int = 10
    gamma_max: float = 1.0
    gamma_scale: float = 5.0
    target_acceptance: float = 0.5
    lambda_init: float = 1.0
    lambda_min: float = -30.0
    sigma2_ratio: float = 1.0
    n_top: int = 20
    n_bottom: int = 50
    m_split: int = 5000
    m_refine: int = 10_000_000
    b_samples: int = 1_000_000
    seed: int = 1
    width: int = 256
    height: int = 256
    max_vertices: int = 20
    metrics_interval: int = 1_000_000
    trace_enabled: bool = False
    dump_partition: bool = False
    # ---- B200 engine knobs ----
    precision: str = "f32"        # "f64" = parity build
    rng: str = "philox"           # "pcg32" = the reference's streams
    adapt_mode: str = "auto"
    lanes_per_chain: int = 0
    device: int = -1
    chains_total: int = 0
    chain_offset: int = 0
    log_steps: int = 0
    steps_per_launch: int = 0
    trace_capacity: int = 0
    region_capacity: int = 0
    b_substreams: int = 0
    profile_kernels: bool = False
    accel: str = "auto"           # "brute" | "bvh"

    def to_c(self) -> _capi.ramlt_render_desc:
        d = _capi.ramlt_render_desc()
        _capi.load().ramlt_gpu_default_desc(C.byref(d))
        for f in fields(self):
            v = getattr(self, f.name)
            if f.name == "strategy":
                v = STRATEGIES[v]
            elif f.name == "perturbation":
                v = PERTURBATIONS[v]
            elif f.name == "precision":
                v = PRECISIONS[v]
            elif f.name == "rng":
                v = RNGS[v]
            elif f.name == "adapt_mode":
                v = ADAPT_MODES[v]
            elif f.name == "accel":
                v = ACCELS[v]
            elif isinstance(v, bool):
                v = int(v)
            setattr(d, f.name, v)
        return d


@dataclass
class RenderResult:
    """ramlt::RenderResult (core/driver.hpp:64-78)."""
    image: np.ndarray
    b: float
    b_stderr: float
    b_samples: int
    total_mutations: int
    perturbation_proposals: int
    large_step_proposals: int
    mean_acceptance: float
    film_luminance: float
    identity_residual: float
    region_count: int
    metrics: np.ndarray                      # (rows, 4): time_s, mutations, rrmse, mean_acc
    trace: np.ndarray                        # (rows, 5): index, region, n, lambda, alpha_hat
    tallies: np.ndarray                      # (regions, 2): accept_sum, visits
    partition_dump: str = ""
    rays_closest: int = 0
    rays_visibility: int = 0
    kernel_launches: int = 0
    extra: dict = field(default_factory=dict)


class Scene:
    """A parsed scene (parse_scene, core/scene.cpp:114-234) owned by the engine library."""

    def __init__(self, text: str, origin: str = "<string>"):
        lib = _capi.load()
        h = C.c_void_p()
        rc = lib.ramlt_scene_parse(text.encode(), origin.encode(), C.byref(h))
        if rc:
            _raise(rc, lib.ramlt_gpu_last_create_error().decode())
        self._h = h
        self.text = text
        self.desc = lib.ramlt_scene_get_desc(h).contents

    @property
    def counts(self):
        d = self.desc
        return d.n_materials, d.n_spheres, d.n_triangles, d.n_emitters

    def __del__(self):
        if getattr(self, "_h", None):
            _capi.load().ramlt_scene_free(self._h)
            self._h = None


def parse_scene(text: str, origin: str = "<string>") -> Scene:
    return Scene(text, origin)


class Engine:
    """One engine handle: one GPU and one chain shard, or -- with ``devices`` --
    every chain over several GPUs of this process (ramlt_gpu_create_multi:
    peer-memory exchanges, film merged every ``film_sync_steps`` lockstep steps)."""

    def __init__(self, scene, cfg: RenderConfig, devices=None, film_sync_steps: int = 4096):
        self.lib = _capi.load()
        self.cfg = cfg
        if isinstance(scene, str):
            scene = Scene(scene)
        self.scene = scene
        self._desc = cfg.to_c()
        h = C.c_void_p()
        if devices is not None:
            devs = (C.c_int32 * max(len(devices), 1))(*devices)
            rc = self.lib.ramlt_gpu_create_multi(C.byref(scene.desc), C.byref(self._desc), len(devices), devs,
                                                 film_sync_steps, C.byref(h))
        else:
            rc = self.lib.ramlt_gpu_create(C.byref(scene.desc), C.byref(self._desc), C.byref(h))
        if rc:
            _raise(rc, self.lib.ramlt_gpu_last_create_error().decode())
        self.h = h

    def _check(self, rc):
        if rc:
            _raise(rc, self.lib.ramlt_gpu_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self.lib.ramlt_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    # --- the span loop -------------------------------------------------------
    def estimate_b(self):
        b, se = C.c_double(), C.c_double()
        self._check(self.lib.ramlt_gpu_estimate_b(self.h, C.byref(b), C.byref(se)))
        return b.value, se.value

    def b_partials(self, begin: int, end: int) -> np.ndarray:
        out = np.zeros((max(end - begin, 0), 2), np.float64)
        self._check(self.lib.ramlt_gpu_estimate_b_partials(
            self.h, begin, end, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def reduce_b(self, partials: np.ndarray):
        p = np.ascontiguousarray(partials, np.float64)
        b, se = C.c_double(), C.c_double()
        self._check(self.lib.ramlt_gpu_reduce_b(self.h, p.ctypes.data_as(C.POINTER(C.c_double)),
                                                p.shape[0], C.byref(b), C.byref(se)))
        return b.value, se.value

    def set_b(self, b: float):
        self._check(self.lib.ramlt_gpu_set_b(self.h, b))

    def init_chains(self):
        self._check(self.lib.ramlt_gpu_init_chains(self.h))

    def run(self, mutations: int):
        self._check(self.lib.ramlt_gpu_run(self.h, mutations))

    def run_steps(self, n: int):
        """Up to n lockstep steps of the canonical span loop (stops at a span
        end); returns (global mutations reached, steps executed)."""
        done, ex = C.c_uint64(), C.c_uint32()
        self._check(self.lib.ramlt_gpu_run_steps(self.h, n, C.byref(done), C.byref(ex)))
        return done.value, ex.value

    def render(self):
        self._check(self.lib.ramlt_gpu_render(self.h))

    def synchronize(self):
        self._check(self.lib.ramlt_gpu_synchronize(self.h))

    # --- outputs -------------------------------------------------------------
    def stats(self) -> _capi.ramlt_stats:
        s = _capi.ramlt_stats()
        self._check(self.lib.ramlt_gpu_read_stats(self.h, C.byref(s)))
        return s

    def film(self):
        """Unscaled fp64 film (H, W, 3) and its total luminance."""
        out = np.zeros((self.cfg.height, self.cfg.width, 3), np.float64)
        lum = C.c_double()
        self._check(self.lib.ramlt_gpu_read_film(self.h, out.ctypes.data_as(C.POINTER(C.c_double)),
                                                 C.byref(lum)))
        return out, lum.value

    def image(self) -> np.ndarray:
        out = np.zeros((self.cfg.height, self.cfg.width, 3), np.float32)
        self._check(self.lib.ramlt_gpu_read_image(self.h, out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def tallies(self) -> np.ndarray:
        n = C.c_uint64()
        self._check(self.lib.ramlt_gpu_read_tallies(self.h, None, None, 0, C.byref(n)))
        acc = np.zeros(n.value, np.float64)
        vis = np.zeros(n.value, np.uint64)
        self._check(self.lib.ramlt_gpu_read_tallies(
            self.h, acc.ctypes.data_as(C.POINTER(C.c_double)),
            vis.ctypes.data_as(C.POINTER(C.c_uint64)), n.value, C.byref(n)))
        return np.stack([acc, vis.astype(np.float64)], axis=1)

    def regions(self):
        n = C.c_uint64()
        self._check(self.lib.ramlt_gpu_read_regions(self.h, None, None, 0, C.byref(n)))
        lam = np.zeros(n.value, np.float64)
        nn = np.zeros(n.value, np.uint64)
        self._check(self.lib.ramlt_gpu_read_regions(
            self.h, lam.ctypes.data_as(C.POINTER(C.c_double)),
            nn.ctypes.data_as(C.POINTER(C.c_uint64)), n.value, C.byref(n)))
        return lam, nn

    def trace(self) -> np.ndarray:
        n = C.c_uint64()
        self._check(self.lib.ramlt_gpu_read_trace(self.h, None, 0, C.byref(n)))
        rows = (_capi.ramlt_trace_row * max(n.value, 1))()
        self._check(self.lib.ramlt_gpu_read_trace(self.h, rows, n.value, C.byref(n)))
        return np.array([[r.mutation_index, r.region, r.n, r.lambda_, r.alpha_hat]
                         for r in rows[: n.value]], np.float64).reshape(-1, 5)

    def metrics(self) -> np.ndarray:
        n = C.c_uint64()
        self._check(self.lib.ramlt_gpu_read_metrics(self.h, None, 0, C.byref(n)))
        out = np.zeros((n.value, 4), np.float64)
        self._check(self.lib.ramlt_gpu_read_metrics(
            self.h, out.ctypes.data_as(C.POINTER(C.c_double)), n.value, C.byref(n)))
        return out

    def decisions(self, K: int):
        a = np.zeros((self.cfg.chains, K), np.float64)
        f = np.zeros((self.cfg.chains, K), np.uint8)
        self._check(self.lib.ramlt_gpu_read_decisions(
            self.h, K, a.ctypes.data_as(C.POINTER(C.c_double)), f.ctypes.data_as(C.POINTER(C.c_uint8))))
        return a, f

    def chain_lengths(self) -> np.ndarray:
        """Current path length k (vertices incl. the camera) of every chain."""
        k = np.zeros(self.cfg.chains, np.int32)
        self._check(self.lib.ramlt_gpu_read_chain_lengths(self.h, k.ctypes.data_as(C.POINTER(C.c_int32))))
        return k

    def partition_dump(self, visits: Optional[np.ndarray] = None) -> str:
        """PartitionIndex::dump; ``visits`` overrides the per-region visit
        counts (sharded runs pass the SUM over ranks)."""
        buf = C.create_string_buffer(1 << 24)
        if visits is None:
            self._check(self.lib.ramlt_gpu_read_partition(self.h, buf, 1 << 24))
        else:
            v = np.ascontiguousarray(visits, np.uint64)
            self._check(self.lib.ramlt_gpu_read_partition_visits(
                self.h, v.ctypes.data_as(C.POINTER(C.c_uint64)), v.size, buf, 1 << 24))
        return buf.value.decode()

    # --- multi-GPU plumbing ------------------------------------------------
    def set_stream(self, stream_ptr: int):
        self._check(self.lib.ramlt_gpu_set_stream(self.h, C.c_void_p(stream_ptr)))

    def film_device(self):
        p = C.POINTER(C.c_double)()
        n = C.c_uint64()
        self._check(self.lib.ramlt_gpu_film_device(self.h, C.byref(p), C.byref(n)))
        return C.cast(p, C.c_void_p).value, n.value

    def adapt_exchange(self):
        c, fx, last = C.POINTER(C.c_uint64)(), C.POINTER(C.c_uint64)(), C.POINTER(C.c_uint64)()
        n = C.c_uint64()
        self._check(self.lib.ramlt_gpu_adapt_exchange(self.h, C.byref(c), C.byref(fx), C.byref(last),
                                                      C.byref(n)))
        cv = lambda p: C.cast(p, C.c_void_p).value  # noqa: E731
        return cv(c), cv(fx), cv(last), n.value

    def adapt_apply(self):
        self._check(self.lib.ramlt_gpu_adapt_apply(self.h))

    def set_exchange_interval(self, steps: int):
        self._check(self.lib.ramlt_gpu_set_exchange_interval(self.h, steps))

    def visits_device(self):
        p = C.POINTER(C.c_uint64)()
        n = C.c_uint64()
        self._check(self.lib.ramlt_gpu_visits_device(self.h, C.byref(p), C.byref(n)))
        return C.cast(p, C.c_void_p).value, n.value

    def refine_pending(self) -> bool:
        f = C.c_int32()
        self._check(self.lib.ramlt_gpu_refine_pending(self.h, C.byref(f)))
        return bool(f.value)

    def refine(self, keep_counts: bool):
        self._check(self.lib.ramlt_gpu_refine(self.h, int(keep_counts)))

    def set_reference(self, image: np.ndarray):
        """RenderConfig::reference (core/driver.hpp:38): metrics rows carry the
        rRMSE of the running image against it (core/driver.cpp:265-272)."""
        img = np.ascontiguousarray(image, np.float32)
        h, w = img.shape[:2]
        self._ref = img
        self._check(self.lib.ramlt_gpu_set_reference(self.h, img.ctypes.data_as(C.POINTER(C.c_float)), w, h))

    def rrmse(self, at: int) -> float:
        """MetricsRow.rrmse (core/driver.cpp:265-272) of the current film at
        ``at`` mutations; NaN without a reference image."""
        out = C.c_double()
        self._check(self.lib.ramlt_gpu_rrmse(self.h, at, C.byref(out)))
        return out.value

    def trace_benchmark(self, n_rays: int):
        """Diagnostic: (kernel ms, hits) of n_rays incoherent closest-hit rays
        through the BVH traversal alone (ramlt_gpu_trace_benchmark)."""
        ms, hits = C.c_double(), C.c_uint64()
        self._check(self.lib.ramlt_gpu_trace_benchmark(self.h, n_rays, C.byref(ms), C.byref(hits)))
        return ms.value, hits.value

    def result(self) -> RenderResult:
        s = self.stats()
        return RenderResult(
            image=self.image(), b=s.b, b_stderr=s.b_stderr, b_samples=s.b_samples,
            total_mutations=s.total_mutations, perturbation_proposals=s.perturbation_proposals,
            large_step_proposals=s.large_step_proposals, mean_acceptance=s.mean_acceptance,
            film_luminance=s.film_luminance, identity_residual=s.identity_residual,
            region_count=s.region_count, metrics=self.metrics(), trace=self.trace(),
            tallies=self.tallies(),
            partition_dump=self.partition_dump() if self.cfg.dump_partition else "",
            rays_closest=s.rays_closest, rays_visibility=s.rays_visibility,
            kernel_launches=s.kernel_launches)


def run_render(scene, cfg: RenderConfig, b: Optional[float] = None,
               reference: Optional[np.ndarray] = None, devices=None,
               film_sync_steps: int = 4096) -> RenderResult:
    """run_render (core/driver.hpp:80): estimate_b, chain init, span loop, reduce.
    ``reference`` is RenderConfig::reference (an (H, W, 3) float32 image);
    ``devices`` (e.g. [0, 1, ..., 7]) runs the chains over several GPUs."""
    eng = Engine(scene, cfg, devices=devices, film_sync_steps=film_sync_steps)
    try:
        if b is not None:
            eng.set_b(b)
        if reference is not None:
            eng.set_reference(reference)
        eng.render()
        return eng.result()
    finally:
        eng.close()

"""ctypes bindings for oracle/_ref (reference harness) and oracle/_build (restatement).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field, fields

import numpy as np

ORACLE_DIR = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libramlt_ref.so")
REF_LOG_SO = os.path.join(ORACLE_DIR, "_ref", "libramlt_ref_log.so")
ORACLE_SO = os.path.join(ORACLE_DIR, "_build", "libramlt_oracle.so")

STRATEGIES = {"fixed": 0, "global": 1, "ra-grid": 2, "ra-quadtree": 3}
PERTURBATIONS = {"lens": 0, "multi-chain": 1}
RNGS = {"pcg32": 0, "philox": 1}
ADAPT_MODES = {"literal": 0, "pooled": 1}


def build(reference: bool = True) -> None:
    """Compile the restatement (always) and the reference harness (when the
    reference sources are present)."""
    target = "all" if reference else "oracle"
    subprocess.run(["make", "-s", "-C", ORACLE_DIR, target, "-j8"], check=True)


class _CConfig(C.Structure):
    _fields_ = [
        ("strategy", C.c_int32), ("perturbation", C.c_int32), ("mutations", C.c_uint64),
        ("chains", C.c_int32), ("batch_size", C.c_int32), ("gamma_max", C.c_double),
        ("gamma_scale", C.c_double), ("target_acceptance", C.c_double),
        ("lambda_init", C.c_double), ("lambda_min", C.c_double), ("sigma2_ratio", C.c_double),
        ("n_top", C.c_int32), ("n_bottom", C.c_int32), ("m_split", C.c_uint64),
        ("m_refine", C.c_uint64), ("b_samples", C.c_uint64), ("seed", C.c_uint64),
        ("width", C.c_int32), ("height", C.c_int32), ("max_vertices", C.c_int32),
        ("trace_enabled", C.c_int32), ("metrics_interval", C.c_uint64),
        ("rng", C.c_int32), ("adapt_mode", C.c_int32), ("b_override", C.c_double),
        ("chain_offset", C.c_int64), ("chains_total", C.c_int64),
    ]


class _CStats(C.Structure):
    _fields_ = [
        ("b", C.c_double), ("b_stderr", C.c_double), ("b_samples", C.c_uint64),
        ("total_mutations", C.c_uint64), ("perturbation_proposals", C.c_uint64),
        ("large_step_proposals", C.c_uint64), ("mean_acceptance", C.c_double),
        ("film_luminance", C.c_double), ("identity_residual", C.c_double),
        ("region_count", C.c_uint64), ("loop_time_s", C.c_double),
        ("rays_closest", C.c_uint64), ("rays_visibility", C.c_uint64),
        ("n_tallies", C.c_uint64), ("n_trace", C.c_uint64), ("n_metrics", C.c_uint64),
    ]


class _CLog(C.Structure):
    _fields_ = [("steps", C.c_uint32), ("a", C.POINTER(C.c_double)),
                ("flags", C.POINTER(C.c_uint8))]


class _CTrace(C.Structure):
    _fields_ = [("mutation_index", C.c_uint64), ("region", C.c_int64), ("n", C.c_uint64),
                ("lambda_", C.c_double), ("alpha_hat", C.c_double)]


class _COutputs(C.Structure):
    _fields_ = [
        ("image", C.POINTER(C.c_float)), ("tally_accept", C.POINTER(C.c_double)),
        ("tally_visits", C.POINTER(C.c_uint64)), ("cap_tallies", C.c_uint64),
        ("trace", C.POINTER(_CTrace)), ("cap_trace", C.c_uint64),
        ("dump", C.c_char_p), ("cap_dump", C.c_uint64),
        ("metrics", C.POINTER(C.c_double)), ("cap_metrics", C.c_uint64),
        ("film", C.POINTER(C.c_double)),
    ]


@dataclass
class OracleConfig:
    """Mirror of ramlt::RenderConfig (core/driver.hpp:19-39) + restatement knobs."""
    strategy: str = "ra-quadtree"
    perturbation: str = "lens"
    mutations: int = 1_000_000
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
    trace_enabled: bool = False
    metrics_interval: int = 1_000_000
    rng: str = "pcg32"
    adapt_mode: str = "literal"
    b_override: float = 0.0
    chain_offset: int = 0
    chains_total: int = 0

    def to_c(self) -> _CConfig:
        c = _CConfig()
        for f in fields(self):
            v = getattr(self, f.name)
            if f.name == "strategy":
                v = STRATEGIES[v]
            elif f.name == "perturbation":
                v = PERTURBATIONS[v]
            elif f.name == "rng":
                v = RNGS[v]
            elif f.name == "adapt_mode":
                v = ADAPT_MODES[v]
            elif f.name == "trace_enabled":
                v = int(bool(v))
            setattr(c, f.name, v)
        return c


@dataclass
class OracleStats:
    b: float = 0.0
    b_stderr: float = 0.0
    b_samples: int = 0
    total_mutations: int = 0
    perturbation_proposals: int = 0
    large_step_proposals: int = 0
    mean_acceptance: float = 0.0
    film_luminance: float = 0.0
    identity_residual: float = 0.0
    region_count: int = 0
    loop_time_s: float = 0.0
    rays_closest: int = 0
    rays_visibility: int = 0


@dataclass
class RenderOutput:
    stats: OracleStats
    image: np.ndarray                        # (H, W, 3) float32, row 0 at the top
    log_a: np.ndarray | None = None          # (chains, K) float64
    log_flags: np.ndarray | None = None      # (chains, K) uint8
    tallies: np.ndarray | None = None        # (R, 2): accept_sum, visits
    trace: np.ndarray | None = None          # (T, 5)
    dump: str = ""
    metrics: np.ndarray | None = None        # (M, 4)
    extra: dict = field(default_factory=dict)

    @property
    def accepted(self) -> np.ndarray:
        return (self.log_flags & 1).astype(bool)

    @property
    def film(self) -> np.ndarray:
        """b-free film: image * N / b (the raw accumulated splat weights)."""
        n = self.stats.total_mutations
        return self.image.astype(np.float64) * (n / self.stats.b) if n else self.image


class RenderError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class _Lib:
    entry = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run oracle.build())")
        self.path = path
        self.lib = C.CDLL(path)
        fn = getattr(self.lib, self.entry)
        fn.restype = C.c_int
        fn.argtypes = [C.c_char_p, C.POINTER(_CConfig), C.POINTER(_CStats), C.POINTER(_CLog),
                       C.POINTER(_COutputs), C.c_char_p, C.c_int]
        self._render = fn

    def render(self, scene: str, cfg: OracleConfig, log_steps: int = 0, cap_tallies: int = 0,
               cap_trace: int = 0, dump: bool = False, cap_metrics: int = 64) -> RenderOutput:
        c = cfg.to_c()
        st = _CStats()
        img = np.zeros((cfg.height, cfg.width, 3), np.float32)
        out = _COutputs()
        out.image = img.ctypes.data_as(C.POINTER(C.c_float))
        ta = np.zeros(max(cap_tallies, 1), np.float64)
        tv = np.zeros(max(cap_tallies, 1), np.uint64)
        out.tally_accept = ta.ctypes.data_as(C.POINTER(C.c_double))
        out.tally_visits = tv.ctypes.data_as(C.POINTER(C.c_uint64))
        out.cap_tallies = cap_tallies
        tr = (_CTrace * max(cap_trace, 1))()
        out.trace = tr
        out.cap_trace = cap_trace
        dbuf = C.create_string_buffer(1 << 22) if dump else None
        out.dump = C.cast(dbuf, C.c_char_p) if dump else None
        out.cap_dump = (1 << 22) if dump else 0
        mt = np.zeros((max(cap_metrics, 1), 4), np.float64)
        film = np.zeros((cfg.height, cfg.width, 3), np.float64)
        out.film = film.ctypes.data_as(C.POINTER(C.c_double))
        out.metrics = mt.ctypes.data_as(C.POINTER(C.c_double))
        out.cap_metrics = cap_metrics
        lg = None
        la = lf = None
        if log_steps:
            la = np.zeros((cfg.chains, log_steps), np.float64)
            lf = np.zeros((cfg.chains, log_steps), np.uint8)
            lg = _CLog(log_steps, la.ctypes.data_as(C.POINTER(C.c_double)),
                       lf.ctypes.data_as(C.POINTER(C.c_uint8)))
        err = C.create_string_buffer(1024)
        rc = self._render(scene.encode(), C.byref(c), C.byref(st), C.byref(lg) if lg else None,
                          C.byref(out), err, 1024)
        if rc != 0:
            raise RenderError(rc, err.value.decode())
        stats = OracleStats(**{f.name: getattr(st, f.name) for f in fields(OracleStats)})
        n_t = min(st.n_tallies, cap_tallies)
        tallies = np.stack([ta[:n_t], tv[:n_t].astype(np.float64)], axis=1) if cap_tallies else None
        n_tr = min(st.n_trace, cap_trace)
        trace = np.array([[tr[i].mutation_index, tr[i].region, tr[i].n, tr[i].lambda_,
                           tr[i].alpha_hat] for i in range(n_tr)], np.float64).reshape(-1, 5)
        return RenderOutput(
            stats=stats, image=img, log_a=la, log_flags=lf, tallies=tallies, trace=trace,
            dump=dbuf.value.decode() if dump else "", metrics=mt[: min(st.n_metrics, cap_metrics)],
            extra={"n_tallies": st.n_tallies, "n_trace": st.n_trace, "film": film})


class RefLib(_Lib):
    """The unmodified reference (oracle/_ref)."""
    entry = "ref_render"

    def __init__(self, log: bool = True):
        super().__init__(REF_LOG_SO if log else REF_SO)
        L = self.lib
        L.ref_normal_quantile.restype = C.c_double
        L.ref_normal_quantile.argtypes = [C.c_double]
        L.ref_normal_cdf.restype = C.c_double
        L.ref_normal_cdf.argtypes = [C.c_double]
        L.ref_angular_pdf.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_double),
                                      C.POINTER(C.c_double)]
        L.ref_angular_sample.argtypes = [C.c_double, C.c_uint64, C.c_uint64, C.c_uint64,
                                         C.POINTER(C.c_double)]
        L.ref_rng_u32.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint32)]
        L.ref_perturb_direction.argtypes = [C.POINTER(C.c_double), C.c_double, C.c_uint64,
                                            C.c_uint64, C.c_uint64, C.POINTER(C.c_double)]
        L.ref_cylindrical.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ref_step_size.restype = C.c_double
        L.ref_step_size.argtypes = [C.c_double, C.c_double, C.c_uint64]
        L.ref_update_lambda.restype = C.c_double
        L.ref_update_lambda.argtypes = [C.c_double, C.c_double, C.c_uint64, C.c_double, C.c_double]
        L.ref_controller_feed.restype = C.c_double
        L.ref_controller_feed.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.POINTER(C.c_int)]
        L.ref_grid_cell.restype = C.c_int
        L.ref_grid_cell.argtypes = [C.c_int, C.c_double, C.c_double]
        L.ref_mh_accept.restype = C.c_double
        L.ref_mh_accept.argtypes = [C.c_double] * 6 + [C.POINTER(C.c_int)]
        L.ref_fresnel.restype = C.c_double
        L.ref_fresnel.argtypes = [C.c_double, C.c_double]
        L.ref_camera.argtypes = [C.POINTER(C.c_double), C.c_int, C.c_int, C.c_double, C.c_double,
                                 C.POINTER(C.c_double), C.POINTER(C.c_double),
                                 C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ref_parse.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.c_char_p, C.c_int]
        L.ref_set_reference.restype = None
        L.ref_set_reference.argtypes = [C.POINTER(C.c_float), C.c_int, C.c_int]
        L.ref_error_report.restype = C.c_int
        L.ref_error_report.argtypes = [C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_int, C.c_int,
                                       C.c_double, C.c_int, C.POINTER(C.c_double)]
        L.ref_autocorrelation_time.restype = C.c_int
        L.ref_autocorrelation_time.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.POINTER(C.c_double),
                                               C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ref_quadtree.restype = C.c_int
        L.ref_quadtree.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.c_uint64, C.c_int,
                                   C.c_char_p, C.c_int]


def ref_set_reference(lib: "RefLib", image):
    """RenderConfig::reference for the next ref_render calls (None clears)."""
    if image is None:
        lib.lib.ref_set_reference(None, 0, 0)
        return
    img = np.ascontiguousarray(image, np.float32)
    lib._ref_keep = img
    lib.lib.ref_set_reference(img.ctypes.data_as(C.POINTER(C.c_float)), img.shape[1], img.shape[0])


def ref_error_report(lib: "RefLib", image, reference, eps: float = 1e-2, rgb: bool = False) -> float:
    a = np.ascontiguousarray(image, np.float32)
    b = np.ascontiguousarray(reference, np.float32)
    out = C.c_double()
    rc = lib.lib.ref_error_report(a.ctypes.data_as(C.POINTER(C.c_float)), b.ctypes.data_as(C.POINTER(C.c_float)),
                                  a.shape[1], a.shape[0], eps, int(rgb), C.byref(out))
    if rc:
        raise RenderError(rc, "error_report: image dimensions differ")
    return out.value


def ref_autocorrelation_time(lib: "RefLib", series):
    """The reference's autocorrelation_time: (tau, n_eff, sigma2), or None where it throws."""
    x = np.ascontiguousarray(series, np.float64)
    t, e, s2 = C.c_double(), C.c_double(), C.c_double()
    rc = lib.lib.ref_autocorrelation_time(x.ctypes.data_as(C.POINTER(C.c_double)), x.size, C.byref(t),
                                          C.byref(e), C.byref(s2))
    return None if rc else (t.value, e.value, s2.value)


def np_autocorrelation_time(series):
    """autocorrelation_time (core/diagnostics.cpp:87-127) in numpy (test checker):
    Geyer's initial positive sequence over rho(k) = sum (x_i - m)(x_{i+k} - m) / (n var)."""
    x = np.asarray(series, np.float64)
    n = x.size
    if n < 1000:
        return None
    m = x.mean()
    var = np.mean((x - m) ** 2)
    if not var > 0:
        return None
    y = x - m
    tau = -1.0
    mm = 0
    while 2 * mm + 1 <= n // 2:
        k0, k1 = 2 * mm, 2 * mm + 1
        g = (np.dot(y[: n - k0], y[k0:]) + np.dot(y[: n - k1], y[k1:])) / (n * var)
        if g <= 0:
            break
        tau += 2 * g
        mm += 1
    tau = max(tau, 1e-3)
    return tau, n / tau, tau / n * var


def np_error_report(image, reference, eps: float = 1e-2) -> float:
    """error_report(..., rgb=false).rrmse (core/diagnostics.cpp:11-38) in numpy (test checker)."""
    a = np.asarray(image, np.float32).astype(np.float64).reshape(-1, 3)
    b = np.asarray(reference, np.float32).astype(np.float64).reshape(-1, 3)
    la = 0.2126 * a[:, 0] + 0.7152 * a[:, 1] + 0.0722 * a[:, 2]
    lb = 0.2126 * b[:, 0] + 0.7152 * b[:, 1] + 0.0722 * b[:, 2]
    e = np.abs(la - lb) / (lb + eps)
    return float(np.sqrt(np.sum(e * e) / e.size))


class OracleLib(_Lib):
    """The restatement (oracle/ramlt_oracle.cpp)."""
    entry = "oracle_render"

    def __init__(self):
        super().__init__(ORACLE_SO)
        L = self.lib
        L.orc_normal_quantile.restype = C.c_double
        L.orc_normal_quantile.argtypes = [C.c_double]
        L.orc_angular_pdf.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_double),
                                      C.POINTER(C.c_double)]
        L.orc_angular_sample.argtypes = [C.c_double, C.c_uint64, C.c_uint64, C.c_uint64,
                                         C.POINTER(C.c_double), C.c_int]
        L.orc_rng_u32.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint32), C.c_int]
        L.orc_philox_block.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                       C.POINTER(C.c_uint32)]
        L.orc_perturb_direction.argtypes = [C.POINTER(C.c_double), C.c_double, C.c_uint64,
                                            C.c_uint64, C.c_uint64, C.POINTER(C.c_double)]
        L.orc_cylindrical.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.orc_update_lambda.restype = C.c_double
        L.orc_update_lambda.argtypes = [C.c_double, C.c_double, C.c_uint64, C.c_double, C.c_double]
        L.orc_grid_cell.restype = C.c_int
        L.orc_grid_cell.argtypes = [C.c_int, C.c_double, C.c_double]
        L.orc_mh_accept.restype = C.c_double
        L.orc_mh_accept.argtypes = [C.c_double] * 6 + [C.POINTER(C.c_int)]
        L.orc_fresnel.restype = C.c_double
        L.orc_fresnel.argtypes = [C.c_double, C.c_double]
        L.orc_b_partials.restype = C.c_int
        L.orc_b_partials.argtypes = [C.c_char_p, C.POINTER(_CConfig), C.c_uint64, C.c_uint64,
                                     C.POINTER(C.c_double)]
        L.orc_camera.argtypes = [C.POINTER(C.c_double), C.c_int, C.c_int, C.c_double, C.c_double,
                                 C.POINTER(C.c_double), C.POINTER(C.c_double),
                                 C.POINTER(C.c_double), C.POINTER(C.c_double)]


def oracle_b_partials(lib: "OracleLib", scene: str, cfg: OracleConfig, begin: int, end: int):
    out = np.zeros((max(end - begin, 0), 2), np.float64)
    c = cfg.to_c()
    rc = lib.lib.orc_b_partials(scene.encode(), C.byref(c), begin, end,
                                out.ctypes.data_as(C.POINTER(C.c_double)))
    if rc:
        raise RenderError(rc, "orc_b_partials failed")
    return out


def dp(arr: np.ndarray):
    return arr.ctypes.data_as(C.POINTER(C.c_double))


# ---- analytic-target harness (BASELINE.json configs[1]) -------------------------------------
MIX_STRATEGIES = {"fixed": 0, "global": 1, "ra-grid": 2}


class _CMixConfig(C.Structure):
    _fields_ = [
        ("strategy", C.c_int32), ("grid_n", C.c_int32), ("chains", C.c_int32),
        ("batch_size", C.c_int32), ("gamma_max", C.c_double), ("gamma_scale", C.c_double),
        ("target_acceptance", C.c_double), ("lambda_init", C.c_double), ("lambda_min", C.c_double),
        ("seed", C.c_uint64), ("steps", C.c_uint64), ("rng", C.c_int32), ("adapt_mode", C.c_int32),
        ("chain_offset", C.c_int64), ("chains_total", C.c_int64), ("log_steps", C.c_uint32),
        ("dim", C.c_int32), ("n_comp", C.c_int32), ("pad_", C.c_int32),
        ("weights", C.POINTER(C.c_double)), ("means", C.POINTER(C.c_double)),
        ("covariances", C.POINTER(C.c_double)),
    ]


class _CMixOut(C.Structure):
    _fields_ = [
        ("x", C.POINTER(C.c_double)), ("log_pi", C.POINTER(C.c_double)),
        ("log_a", C.POINTER(C.c_double)), ("log_f", C.POINTER(C.c_uint8)),
        ("lambda_", C.POINTER(C.c_double)), ("n", C.POINTER(C.c_uint64)),
        ("tally_accept", C.POINTER(C.c_double)), ("tally_visits", C.POINTER(C.c_uint64)),
        ("cap_regions", C.c_uint64), ("trace", C.POINTER(_CTrace)), ("cap_trace", C.c_uint64),
        ("n_trace", C.c_uint64), ("n_regions", C.c_uint64), ("accepted", C.c_uint64),
        ("acceptance_sum", C.c_double),
    ]


@dataclass
class OracleMixConfig:
    strategy: str = "global"
    grid_n: int = 4
    chains: int = 1
    batch_size: int = 10
    gamma_max: float = 1.0
    gamma_scale: float = 5.0
    target_acceptance: float = 0.5
    lambda_init: float = 1.0
    lambda_min: float = -30.0
    seed: int = 1
    steps: int = 16
    rng: str = "pcg32"
    adapt_mode: str = "literal"
    chain_offset: int = 0
    chains_total: int = 0
    log_steps: int = 0


def mix_run(target, cfg: OracleMixConfig, reference: bool = False, cap_trace: int = 1 << 16) -> dict:
    """Run the analytic-target chain loop on the CPU: the restatement
    (oracle_mix_run) or the reference composition (ref_mix_run, PCG32 +
    literal lockstep only).  ``target`` is a paper_2402_08273_b200.mix.MixTarget
    (or anything with weights / means / covariances arrays)."""
    path = REF_SO if reference else ORACLE_SO
    lib = C.CDLL(path)
    fn = getattr(lib, "ref_mix_run" if reference else "oracle_mix_run")
    fn.restype = C.c_int
    fn.argtypes = [C.POINTER(_CMixConfig), C.POINTER(_CMixOut), C.c_char_p, C.c_int]
    w = np.ascontiguousarray(target.weights, np.float64)
    mu = np.ascontiguousarray(target.means, np.float64)
    cov = np.ascontiguousarray(target.covariances, np.float64)
    K, D = mu.shape
    c = _CMixConfig()
    for f in fields(cfg):
        v = getattr(cfg, f.name)
        if f.name == "strategy":
            v = MIX_STRATEGIES[v]
        elif f.name == "rng":
            v = RNGS[v]
        elif f.name == "adapt_mode":
            v = ADAPT_MODES[v]
        setattr(c, f.name, v)
    c.dim, c.n_comp = D, K
    c.weights, c.means, c.covariances = dp(w), dp(mu), dp(cov)
    nreg = cfg.grid_n * cfg.grid_n if cfg.strategy == "ra-grid" else 1
    x = np.zeros((cfg.chains, D))
    lp = np.zeros(cfg.chains)
    L = max(cfg.log_steps, 1)
    la = np.zeros((cfg.chains, L))
    lf = np.zeros((cfg.chains, L), np.uint8)
    lam, acc = np.zeros(nreg), np.zeros(nreg)
    n, vis = np.zeros(nreg, np.uint64), np.zeros(nreg, np.uint64)
    tr = (_CTrace * max(cap_trace, 1))()
    o = _CMixOut()
    o.x, o.log_pi, o.log_a = dp(x), dp(lp), dp(la)
    o.log_f = lf.ctypes.data_as(C.POINTER(C.c_uint8))
    o.lambda_, o.tally_accept = dp(lam), dp(acc)
    o.n = n.ctypes.data_as(C.POINTER(C.c_uint64))
    o.tally_visits = vis.ctypes.data_as(C.POINTER(C.c_uint64))
    o.cap_regions = nreg
    o.trace, o.cap_trace = tr, cap_trace
    err = C.create_string_buffer(1024)
    rc = fn(C.byref(c), C.byref(o), err, 1024)
    if rc:
        raise RenderError(rc, err.value.decode())
    nt = min(o.n_trace, cap_trace)
    trace = np.array([[tr[i].mutation_index, tr[i].region, tr[i].n, tr[i].lambda_, tr[i].alpha_hat]
                      for i in range(nt)], np.float64).reshape(-1, 5)
    props = cfg.chains * cfg.steps
    return dict(x=x, log_pi=lp, log_a=la[:, : cfg.log_steps], log_f=lf[:, : cfg.log_steps],
                lambda_=lam, n=n, tally_accept=acc, tally_visits=vis, trace=trace,
                accepted=o.accepted, acceptance_sum=o.acceptance_sum,
                mean_acceptance=o.acceptance_sum / props if props else 0.0)

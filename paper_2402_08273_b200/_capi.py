"""ctypes binding of libramlt_gpu.so (include/ramlt_gpu.h).

The product path: there is no CPU fallback.  If the in-tree CUDA library is
missing, importing the engine raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RAMLT_GPU_LIB") or os.path.join(PKG_DIR, "_lib", "libramlt_gpu.so")


class ramlt_material(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("albedo", C.c_double * 3),
                ("ior", C.c_double), ("exponent", C.c_double)]


class ramlt_sphere(C.Structure):
    _fields_ = [("center", C.c_double * 3), ("radius", C.c_double), ("material", C.c_int32),
                ("emitter", C.c_int32)]


class ramlt_triangle(C.Structure):
    _fields_ = [("a", C.c_double * 3), ("b", C.c_double * 3), ("c", C.c_double * 3),
                ("material", C.c_int32), ("emitter", C.c_int32)]


class ramlt_scene_desc(C.Structure):
    _fields_ = [("cam_position", C.c_double * 3), ("cam_look_at", C.c_double * 3),
                ("cam_up", C.c_double * 3), ("cam_fov_deg", C.c_double),
                ("n_materials", C.c_int32), ("n_spheres", C.c_int32),
                ("n_triangles", C.c_int32), ("n_emitters", C.c_int32),
                ("materials", C.POINTER(ramlt_material)), ("spheres", C.POINTER(ramlt_sphere)),
                ("triangles", C.POINTER(ramlt_triangle)),
                ("emitter_radiance", C.POINTER(C.c_double))]


class ramlt_render_desc(C.Structure):
    _fields_ = [
        ("strategy", C.c_int32), ("perturbation", C.c_int32), ("mutations", C.c_uint64),
        ("time_budget_s", C.c_double), ("chains", C.c_int32), ("batch_size", C.c_int32),
        ("gamma_max", C.c_double), ("gamma_scale", C.c_double),
        ("target_acceptance", C.c_double), ("lambda_init", C.c_double),
        ("lambda_min", C.c_double), ("sigma2_ratio", C.c_double), ("n_top", C.c_int32),
        ("n_bottom", C.c_int32), ("m_split", C.c_uint64), ("m_refine", C.c_uint64),
        ("b_samples", C.c_uint64), ("seed", C.c_uint64), ("width", C.c_int32),
        ("height", C.c_int32), ("max_vertices", C.c_int32), ("trace_enabled", C.c_int32),
        ("metrics_interval", C.c_uint64), ("dump_partition", C.c_int32),
        ("precision", C.c_int32), ("rng", C.c_int32), ("adapt_mode", C.c_int32),
        ("lanes_per_chain", C.c_int32), ("device", C.c_int32), ("pad_", C.c_int32),
        ("chains_total", C.c_int64), ("chain_offset", C.c_int64), ("log_steps", C.c_uint32),
        ("steps_per_launch", C.c_uint32), ("trace_capacity", C.c_uint64),
        ("region_capacity", C.c_uint64), ("b_substreams", C.c_uint64),
        ("profile_kernels", C.c_int32), ("accel", C.c_int32),
    ]


class ramlt_stats(C.Structure):
    _fields_ = [
        ("b", C.c_double), ("b_stderr", C.c_double), ("b_samples", C.c_uint64),
        ("total_mutations", C.c_uint64), ("perturbation_proposals", C.c_uint64),
        ("large_step_proposals", C.c_uint64), ("mean_acceptance", C.c_double),
        ("film_luminance", C.c_double), ("identity_residual", C.c_double),
        ("region_count", C.c_uint64), ("loop_time_s", C.c_double),
        ("rays_closest", C.c_uint64), ("rays_visibility", C.c_uint64),
        ("n_tallies", C.c_uint64), ("n_trace", C.c_uint64), ("n_metrics", C.c_uint64),
        ("kernel_launches", C.c_uint64), ("step_kernel_ms", C.c_double),
        ("step_kernel_launches", C.c_uint64), ("trace_kernel_ms", C.c_double),
        ("trace_kernel_launches", C.c_uint64), ("wavefront_rounds", C.c_uint64),
    ]


class ramlt_trace_row(C.Structure):
    _fields_ = [("mutation_index", C.c_uint64), ("region", C.c_int64), ("n", C.c_uint64),
                ("lambda_", C.c_double), ("alpha_hat", C.c_double)]


class ramlt_mix_target(C.Structure):
    _fields_ = [("dim", C.c_int32), ("n_comp", C.c_int32), ("weights", C.POINTER(C.c_double)),
                ("means", C.POINTER(C.c_double)), ("covariances", C.POINTER(C.c_double))]


class ramlt_mix_desc(C.Structure):
    _fields_ = [
        ("strategy", C.c_int32), ("grid_n", C.c_int32), ("chains", C.c_int32),
        ("batch_size", C.c_int32), ("gamma_max", C.c_double), ("gamma_scale", C.c_double),
        ("target_acceptance", C.c_double), ("lambda_init", C.c_double),
        ("lambda_min", C.c_double), ("seed", C.c_uint64), ("precision", C.c_int32),
        ("rng", C.c_int32), ("adapt_mode", C.c_int32), ("device", C.c_int32),
        ("chains_total", C.c_int64), ("chain_offset", C.c_int64), ("log_steps", C.c_uint32),
        ("trace_enabled", C.c_int32), ("trace_capacity", C.c_uint64),
        ("profile_kernels", C.c_int32), ("cooperative", C.c_int32),
        ("series_steps", C.c_uint32), ("series_dim", C.c_int32),
    ]


class ramlt_mix_stats(C.Structure):
    _fields_ = [
        ("steps", C.c_uint64), ("proposals", C.c_uint64), ("accepted", C.c_uint64),
        ("acceptance_sum", C.c_double), ("mean_acceptance", C.c_double),
        ("region_count", C.c_uint64), ("n_trace", C.c_uint64), ("kernel_launches", C.c_uint64),
        ("step_kernel_ms", C.c_double), ("step_kernel_launches", C.c_uint64),
    ]


P = C.POINTER
vp = C.c_void_p
H = C.c_void_p  # opaque ramlt_gpu*

# name -> (restype, argtypes); also the exported-symbol list the CPU tests check
SIGNATURES = {
    "ramlt_gpu_abi_version": (C.c_int, []),
    "ramlt_gpu_default_desc": (None, [P(ramlt_render_desc)]),
    "ramlt_scene_parse": (C.c_int, [C.c_char_p, C.c_char_p, P(vp)]),
    "ramlt_scene_get_desc": (P(ramlt_scene_desc), [vp]),
    "ramlt_scene_free": (None, [vp]),
    "ramlt_gpu_create": (C.c_int, [P(ramlt_scene_desc), P(ramlt_render_desc), P(H)]),
    "ramlt_gpu_create_from_text": (C.c_int, [C.c_char_p, C.c_char_p, P(ramlt_render_desc), P(H)]),
    "ramlt_gpu_create_multi": (C.c_int, [P(ramlt_scene_desc), P(ramlt_render_desc), C.c_int32, P(C.c_int32),
                                         C.c_uint32, P(H)]),
    "ramlt_gpu_create_multi_from_text": (C.c_int, [C.c_char_p, C.c_char_p, P(ramlt_render_desc), C.c_int32,
                                                   P(C.c_int32), C.c_uint32, P(H)]),
    "ramlt_gpu_last_create_error": (C.c_char_p, []),
    "ramlt_gpu_estimate_b": (C.c_int, [H, P(C.c_double), P(C.c_double)]),
    "ramlt_gpu_estimate_b_partials": (C.c_int, [H, C.c_uint64, C.c_uint64, P(C.c_double)]),
    "ramlt_gpu_reduce_b": (C.c_int, [H, P(C.c_double), C.c_uint64, P(C.c_double), P(C.c_double)]),
    "ramlt_gpu_set_b": (C.c_int, [H, C.c_double]),
    "ramlt_gpu_init_chains": (C.c_int, [H]),
    "ramlt_gpu_run": (C.c_int, [H, C.c_uint64]),
    "ramlt_gpu_run_steps": (C.c_int, [H, C.c_uint32, P(C.c_uint64), P(C.c_uint32)]),
    "ramlt_gpu_render": (C.c_int, [H]),
    "ramlt_gpu_synchronize": (C.c_int, [H]),
    "ramlt_gpu_read_stats": (C.c_int, [H, P(ramlt_stats)]),
    "ramlt_gpu_read_film": (C.c_int, [H, P(C.c_double), P(C.c_double)]),
    "ramlt_gpu_read_image": (C.c_int, [H, P(C.c_float)]),
    "ramlt_gpu_read_tallies": (C.c_int, [H, P(C.c_double), P(C.c_uint64), C.c_uint64, P(C.c_uint64)]),
    "ramlt_gpu_read_regions": (C.c_int, [H, P(C.c_double), P(C.c_uint64), C.c_uint64, P(C.c_uint64)]),
    "ramlt_gpu_read_trace": (C.c_int, [H, P(ramlt_trace_row), C.c_uint64, P(C.c_uint64)]),
    "ramlt_gpu_read_metrics": (C.c_int, [H, P(C.c_double), C.c_uint64, P(C.c_uint64)]),
    "ramlt_gpu_read_decisions": (C.c_int, [H, C.c_uint32, P(C.c_double), P(C.c_uint8)]),
    "ramlt_gpu_read_partition": (C.c_int, [H, C.c_char_p, C.c_uint64]),
    "ramlt_gpu_read_partition_visits": (C.c_int, [H, P(C.c_uint64), C.c_uint64, C.c_char_p, C.c_uint64]),
    "ramlt_gpu_read_chain_lengths": (C.c_int, [H, P(C.c_int32)]),
    "ramlt_gpu_set_stream": (C.c_int, [H, vp]),
    "ramlt_gpu_film_device": (C.c_int, [H, P(P(C.c_double)), P(C.c_uint64)]),
    "ramlt_gpu_adapt_exchange": (C.c_int, [H, P(P(C.c_uint64)), P(P(C.c_uint64)),
                                           P(P(C.c_uint64)), P(C.c_uint64)]),
    "ramlt_gpu_adapt_apply": (C.c_int, [H]),
    "ramlt_gpu_set_exchange_interval": (C.c_int, [H, C.c_uint32]),
    "ramlt_gpu_visits_device": (C.c_int, [H, P(P(C.c_uint64)), P(C.c_uint64)]),
    "ramlt_gpu_refine_pending": (C.c_int, [H, P(C.c_int32)]),
    "ramlt_gpu_refine": (C.c_int, [H, C.c_int32]),
    "ramlt_gpu_set_reference": (C.c_int, [H, P(C.c_float), C.c_int32, C.c_int32]),
    "ramlt_gpu_rrmse": (C.c_int, [H, C.c_uint64, P(C.c_double)]),
    "ramlt_gpu_trace_benchmark": (C.c_int, [H, C.c_uint64, P(C.c_double), P(C.c_uint64)]),
    "ramlt_gpu_last_error": (C.c_char_p, [H]),
    "ramlt_gpu_destroy": (None, [H]),
    # include/ramlt_mix.h -- analytic-target adaptive MCMC (BASELINE.json configs[1])
    "ramlt_mix_default_desc": (None, [P(ramlt_mix_desc)]),
    "ramlt_mix_create": (C.c_int, [P(ramlt_mix_target), P(ramlt_mix_desc), P(H)]),
    "ramlt_mix_last_create_error": (C.c_char_p, []),
    "ramlt_mix_last_error": (C.c_char_p, [H]),
    "ramlt_mix_destroy": (None, [H]),
    "ramlt_mix_set_stream": (C.c_int, [H, vp]),
    "ramlt_mix_init_chains": (C.c_int, [H]),
    "ramlt_mix_run": (C.c_int, [H, C.c_uint64]),
    "ramlt_mix_synchronize": (C.c_int, [H]),
    "ramlt_mix_read_stats": (C.c_int, [H, P(ramlt_mix_stats)]),
    "ramlt_mix_read_state": (C.c_int, [H, P(C.c_double), P(C.c_double)]),
    "ramlt_mix_read_chain_tallies": (C.c_int, [H, P(C.c_double), P(C.c_uint64)]),
    "ramlt_mix_read_regions": (C.c_int, [H, P(C.c_double), P(C.c_uint64), P(C.c_double),
                                         P(C.c_uint64), C.c_uint64, P(C.c_uint64)]),
    "ramlt_mix_read_trace": (C.c_int, [H, P(ramlt_trace_row), C.c_uint64, P(C.c_uint64)]),
    "ramlt_mix_read_decisions": (C.c_int, [H, C.c_uint32, P(C.c_double), P(C.c_uint8)]),
    "ramlt_mix_read_series": (C.c_int, [H, P(C.c_double)]),
    "ramlt_mix_autocorrelation": (C.c_int, [H, C.c_int32, C.c_int32, P(C.c_double), P(C.c_double),
                                            P(C.c_double), P(C.c_int32)]),
    "ramlt_mix_adapt_exchange": (C.c_int, [H, P(P(C.c_uint64)), P(P(C.c_uint64)),
                                           P(P(C.c_uint64)), P(C.c_uint64)]),
    "ramlt_mix_adapt_apply": (C.c_int, [H]),
    "ramlt_mix_set_external_adaptation": (C.c_int, [H, C.c_int]),
}

_lib = None


def load() -> C.CDLL:
    """Load the in-tree CUDA library; raise loudly when it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: the B200 engine has no CPU fallback. "
                "Build it with `python -c 'import __graft_entry__ as g; g.build()'`.")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib

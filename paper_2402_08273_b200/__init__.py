"""B200-native (sm_100a) data-parallel hot path of regional adaptive Metropolis
light transport (arXiv 2402.08273): the per-chain mutation step behind the
reference's ``run_render`` (core/driver.hpp:80), as hand-written CUDA kernels
behind a C-ABI (include/ramlt_gpu.h).

The CUDA library is loaded lazily on first use and there is no CPU fallback.
"""
from .render import (  # noqa: F401
    RenderConfig, RenderResult, Engine, Scene, parse_scene, run_render, LogicError, CudaError,
)
from . import scenes  # noqa: F401

__all__ = ["RenderConfig", "RenderResult", "Engine", "Scene", "parse_scene", "run_render",
           "LogicError", "CudaError", "scenes"]

"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the build container (needs /root/reference to build oracle/_ref):
    python tests/golden/make_golden.py
Each fixture stores the scene text, the config, and the reference's outputs:
per-chain decision logs (a, flags) of the first K steps, the image, b, result
scalars, tallies, adaptation trace and partition dump.  Fixed-strategy cases
are deterministic at any chain count; adaptive cases use one chain, where the
reference is deterministic.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.abi import OracleConfig, RefLib, build  # noqa: E402
from paper_2402_08273_b200 import scenes  # noqa: E402

K = 32

CASES = [
    # name, scene, config overrides
    ("c1_fixed_lens", "cornell", dict(strategy="fixed", perturbation="lens", chains=64,
                                      mutations=64 * 48, max_vertices=9)),
    ("c1_fixed_lens_s2", "cornell", dict(strategy="fixed", perturbation="lens", chains=64,
                                         mutations=64 * 48, max_vertices=9, seed=2)),
    ("c1_fixed_lens_ragged", "cornell", dict(strategy="fixed", perturbation="lens", chains=48,
                                             mutations=1000, max_vertices=9, metrics_interval=333,
                                             m_refine=500)),
    ("c1_global_lens_1c", "cornell", dict(strategy="global", perturbation="lens", chains=1,
                                          mutations=3000, max_vertices=9, trace_enabled=True)),
    ("c1_ragrid_lens_1c", "cornell", dict(strategy="ra-grid", perturbation="lens", chains=1,
                                          mutations=3000, max_vertices=9, trace_enabled=True)),
    ("c1_raquad_lens_1c", "cornell", dict(strategy="ra-quadtree", perturbation="lens", chains=1,
                                          mutations=4000, max_vertices=9, trace_enabled=True,
                                          m_refine=1000, m_split=150)),
    ("c3_fixed_mc", "caustic", dict(strategy="fixed", perturbation="multi-chain", chains=64,
                                    mutations=64 * 48, max_vertices=17)),
    ("c3_raquad_mc_1c", "caustic", dict(strategy="ra-quadtree", perturbation="multi-chain", chains=1,
                                        mutations=4000, max_vertices=17, trace_enabled=True,
                                        m_refine=1000, m_split=100, n_top=4, seed=3)),
    ("mix_fixed_mc", "mirror", dict(strategy="fixed", perturbation="multi-chain", chains=64,
                                    mutations=64 * 48, max_vertices=12)),
    ("mix_fixed_lens", "mirror", dict(strategy="fixed", perturbation="lens", chains=64,
                                      mutations=64 * 48, max_vertices=12)),
    ("mix_ragrid_mc_1c", "mirror", dict(strategy="ra-grid", perturbation="multi-chain", chains=1,
                                        mutations=3000, max_vertices=12, trace_enabled=True,
                                        n_top=4, n_bottom=5, seed=2)),
    ("mix_global_mc_1c", "mirror", dict(strategy="global", perturbation="multi-chain", chains=1,
                                        mutations=3000, max_vertices=12, trace_enabled=True, seed=2)),
]


def run_case(ref: RefLib, name: str, scene_name: str, over: dict) -> dict:
    scene = scenes.SCENES[scene_name]()
    base = dict(width=64, height=64, b_samples=20000, seed=1, metrics_interval=1_000_000)
    base.update(over)
    cfg = OracleConfig(**base)
    k = K if cfg.chains > 1 else int(cfg.mutations)
    out = ref.render(scene, cfg, log_steps=k, cap_tallies=1 << 16, cap_trace=1 << 16, dump=True)
    s = out.stats
    return dict(
        name=name, scene=scene, config=json.dumps(base),
        log_a=out.log_a, log_flags=out.log_flags, image=out.image,
        stats=np.array([s.b, s.b_stderr, s.total_mutations, s.perturbation_proposals,
                        s.large_step_proposals, s.mean_acceptance, s.film_luminance,
                        s.identity_residual, s.region_count, s.rays_closest, s.rays_visibility],
                       np.float64),
        tallies=out.tallies, trace=out.trace, dump=out.dump, metrics=out.metrics)


STAT_KEYS = ["b", "b_stderr", "total_mutations", "perturbation_proposals", "large_step_proposals",
             "mean_acceptance", "film_luminance", "identity_residual", "region_count",
             "rays_closest", "rays_visibility"]


def kat_values(ref: RefLib) -> dict:
    """SPEC known-answer values evaluated by the reference's own functions."""
    import ctypes as C
    L = ref.lib
    pdf, pdf_sa = C.c_double(), C.c_double()
    L.ref_angular_pdf(1.0, 0.0, C.byref(pdf), C.byref(pdf_sa))
    st = C.c_int()
    cam = (C.c_double * 10)(0.5, 0.5, -1.0, 0.5, 0.5, 0.5, 0.0, 1.0, 0.0, 45.0)
    d3, uv, imp, dp = (C.c_double * 3)(), (C.c_double * 2)(), C.c_double(), C.c_double()
    L.ref_camera(cam, 256, 256, 0.3, 0.7, d3, uv, C.byref(imp), C.byref(dp))
    w = (C.c_double * 3)(1.0, 0.0, 0.0)
    cy = (C.c_double * 2)()
    L.ref_cylindrical(w, cy)
    u32 = (C.c_uint32 * 16)()
    L.ref_rng_u32(1, 0, 16, u32)
    u32b = (C.c_uint32 * 16)()
    L.ref_rng_u32(42, 0x4000000000000001, 16, u32b)
    return {
        "angular_pdf0_sigma1": pdf.value,
        "sigma_lambda1": float(np.exp(0.5)),
        "step_size_100": L.ref_step_size(1.0, 5.0, 100),
        "update_lambda_1_0.3": L.ref_update_lambda(1.0, 0.3, 1, 0.5, -30.0),
        "update_lambda_clamp": L.ref_update_lambda(-30.0, 0.1, 1, 0.5, -30.0),
        "grid20_center": L.ref_grid_cell(20, 0.5, 0.5),
        "grid20_corner": L.ref_grid_cell(20, 1.0, 1.0),
        "mh_equal": L.ref_mh_accept(1.0, 1.0, 1.0, 1.0, 0.5, 0.5, C.byref(st)),
        "mh_double": L.ref_mh_accept(1.0, 2.0, 1.0, 1.0, 0.5, 0.5, C.byref(st)),
        "fresnel_normal_1.5": L.ref_fresnel(1.0, 1.5),
        "camera_dir": list(d3), "camera_uv": list(uv), "camera_importance": imp.value,
        "camera_dir_pdf": dp.value, "cylindrical_x": list(cy),
        "pcg_seed1_stream0": list(u32), "pcg_seed42_init": list(u32b),
        "normal_quantile": [L.ref_normal_quantile(p) for p in (1e-10, 0.01, 0.3, 0.5, 0.9, 0.99999)],
    }


def main() -> None:
    build(reference=True)
    ref = RefLib(log=True)
    for name, scene, over in CASES:
        d = run_case(ref, name, scene, over)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)
        st = dict(zip(STAT_KEYS, d["stats"].tolist()))
        print(name, "acc=%.4f" % st["mean_acceptance"], "accepted=%d" % int((d["log_flags"] & 1).sum()),
              "pert=%d" % int(((d["log_flags"] >> 1) & 1).sum()), "regions=%d" % st["region_count"],
              "trace=%d" % len(d["trace"]))
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat_values(ref), f, indent=1)


if __name__ == "__main__":
    main()

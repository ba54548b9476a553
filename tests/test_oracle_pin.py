"""Pins the restatement oracle (oracle/ramlt_oracle.cpp) to the UNMODIFIED
reference: against the committed golden fixtures (generated from the reference
by tests/golden/make_golden.py) and, when the reference harness is built in
this container, against live reference runs on fresh seeds.  Bar: bit-exact."""
import ctypes as C
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, GOLDEN_CASES, golden_stats, load_golden


def oracle_run(lib, g, **over):
    from oracle.abi import OracleConfig
    cfg = OracleConfig(**dict(g["config"], **over))
    cfg.b_override = golden_stats(g)["b"]
    K = g["log_a"].shape[1]
    return lib.render(g["scene"], cfg, log_steps=K, cap_tallies=1 << 16, cap_trace=1 << 16, dump=True)


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_oracle_matches_reference_golden(name, oracle_lib):
    g = load_golden(name)
    st = golden_stats(g)
    o = oracle_run(oracle_lib, g)
    assert np.array_equal(o.log_flags, g["log_flags"])
    assert np.array_equal(o.log_a, g["log_a"])          # bit-exact
    assert np.array_equal(o.image, g["image"])          # bit-exact film (b from the golden)
    s = o.stats
    assert s.total_mutations == st["total_mutations"]
    assert s.perturbation_proposals == st["perturbation_proposals"]
    assert s.large_step_proposals == st["large_step_proposals"]
    assert s.mean_acceptance == st["mean_acceptance"]
    assert s.film_luminance == st["film_luminance"]
    assert s.region_count == st["region_count"]
    assert s.rays_closest == st["rays_closest"]
    assert s.rays_visibility == st["rays_visibility"]
    assert s.identity_residual == st["identity_residual"]
    assert np.array_equal(o.tallies[: len(g["tallies"])], g["tallies"])
    assert np.array_equal(o.trace, g["trace"])
    assert o.dump == g["dump"]
    # Film luminance sums to the mutation count
    assert s.film_luminance == pytest.approx(s.total_mutations, rel=1e-9)
    # Appendix-B identity
    assert s.identity_residual <= 1e-12


@pytest.mark.parametrize("seed", [11, 12])
@pytest.mark.parametrize("scene_name,pert,strategy,chains", [
    ("cornell", "lens", "fixed", 24), ("caustic", "multi-chain", "fixed", 24),
    ("mirror", "lens", "ra-quadtree", 1), ("mirror", "multi-chain", "ra-grid", 1),
])
def test_oracle_matches_reference_live(ref_lib, oracle_lib, seed, scene_name, pert, strategy, chains):
    from oracle.abi import OracleConfig
    from paper_2402_08273_b200 import scenes
    scene = scenes.SCENES[scene_name]()
    cfg = OracleConfig(strategy=strategy, perturbation=pert, chains=chains, mutations=chains * 40 + 7,
                       width=48, height=40, max_vertices=14, b_samples=5000, seed=seed,
                       trace_enabled=True, m_refine=500, m_split=60, n_top=3, n_bottom=4)
    r = ref_lib.render(scene, cfg, log_steps=40, cap_tallies=4096, cap_trace=4096, dump=True)
    cfg.b_override = r.stats.b
    o = oracle_lib.render(scene, cfg, log_steps=40, cap_tallies=4096, cap_trace=4096, dump=True)
    assert np.array_equal(r.log_flags, o.log_flags)
    assert np.array_equal(r.log_a, o.log_a)
    assert np.array_equal(r.image, o.image)
    assert np.array_equal(r.trace, o.trace)
    assert r.dump == o.dump
    assert r.stats.rays_closest == o.stats.rays_closest


def test_edge_cases_oracle_vs_reference(ref_lib, oracle_lib):
    """Zero-mutation budget (black film), max_vertices = 2 (camera -> light only),
    chains > mutations (ragged spans), and the error contracts."""
    from oracle.abi import OracleConfig, RenderError
    from paper_2402_08273_b200 import scenes
    scene = scenes.cornell_box()
    for over in (dict(mutations=0, chains=3), dict(max_vertices=2, chains=4, mutations=50),
                 dict(chains=10, mutations=7), dict(chains=5, mutations=23, metrics_interval=4,
                                                    m_refine=6, strategy="ra-quadtree", m_split=1)):
        cfg = OracleConfig(**dict(dict(strategy="fixed", perturbation="lens", width=16, height=16,
                                       max_vertices=9, b_samples=3000, seed=5), **over))
        r = ref_lib.render(scene, cfg, log_steps=8, cap_tallies=256, dump=True)
        cfg.b_override = r.stats.b
        o = oracle_lib.render(scene, cfg, log_steps=8, cap_tallies=256, dump=True)
        assert np.array_equal(r.log_flags, o.log_flags), over
        assert np.array_equal(r.image, o.image), over
        assert r.stats.total_mutations == o.stats.total_mutations
        assert r.dump == o.dump, over
    # error contracts: chains < 1 (logic_error), black scene (runtime_error)
    for lib in (ref_lib, oracle_lib):
        with pytest.raises(RenderError) as e:
            lib.render(scene, OracleConfig(chains=0, mutations=1, b_samples=10))
        assert e.value.code == 2
    black = scene.replace("emitter 34 17.0 12.0 4.0", "emitter 34 0.0 0.0 0.0").replace(
        "emitter 35 17.0 12.0 4.0", "emitter 35 0.0 0.0 0.0")
    for lib in (ref_lib, oracle_lib):
        with pytest.raises(RenderError) as e:
            lib.render(black, OracleConfig(chains=1, mutations=1, b_samples=100, width=8, height=8))
        assert e.value.code == 1 and "black-scene" in str(e.value)


def test_kat_values_from_reference(oracle_lib):
    """SPEC known answers evaluated by the
    reference (kat.json) and reproduced by the oracle."""
    kat = json.load(open(os.path.join(GOLDEN, "kat.json")))
    L = oracle_lib.lib
    assert kat["angular_pdf0_sigma1"] == pytest.approx(0.399615, abs=1e-5)
    pdf, sa = C.c_double(), C.c_double()
    L.orc_angular_pdf(1.0, 0.0, C.byref(pdf), C.byref(sa))
    assert pdf.value == kat["angular_pdf0_sigma1"]
    assert kat["sigma_lambda1"] == pytest.approx(1.648721, abs=1e-6)
    assert kat["step_size_100"] == 0.5
    assert kat["update_lambda_1_0.3"] == 0.0 == L.orc_update_lambda(1.0, 0.3, 1, 0.5, -30.0)
    assert kat["update_lambda_clamp"] == -30.0 == L.orc_update_lambda(-30.0, 0.1, 1, 0.5, -30.0)
    assert kat["grid20_center"] == 210 == L.orc_grid_cell(20, 0.5, 0.5)
    assert kat["grid20_corner"] == 399 == L.orc_grid_cell(20, 1.0, 1.0)
    st = C.c_int()
    assert kat["mh_equal"] == 1.0 == L.orc_mh_accept(1.0, 1.0, 1.0, 1.0, 0.5, 0.5, C.byref(st))
    assert kat["mh_double"] == 1.0 == L.orc_mh_accept(1.0, 2.0, 1.0, 1.0, 0.5, 0.5, C.byref(st))
    L.orc_mh_accept(0.0, 1.0, 1.0, 1.0, 0.5, 0.5, C.byref(st))
    assert st.value == 3   # zero-measure current state throws std::invalid_argument
    assert kat["fresnel_normal_1.5"] == pytest.approx(0.04) and L.orc_fresnel(1.0, 1.5) == kat["fresnel_normal_1.5"]
    cam = (C.c_double * 10)(0.5, 0.5, -1.0, 0.5, 0.5, 0.5, 0.0, 1.0, 0.0, 45.0)
    d3, uv, imp, dp = (C.c_double * 3)(), (C.c_double * 2)(), C.c_double(), C.c_double()
    L.orc_camera(cam, 256, 256, 0.3, 0.7, d3, uv, C.byref(imp), C.byref(dp))
    assert list(d3) == kat["camera_dir"] and imp.value == kat["camera_importance"]
    assert dp.value == kat["camera_dir_pdf"]
    assert abs(uv[0] - 0.3) < 1e-9 and abs(uv[1] - 0.7) < 1e-9   # SPEC.md:70 round trip
    w = (C.c_double * 3)(1.0, 0.0, 0.0)
    cy = (C.c_double * 2)()
    L.orc_cylindrical(w, cy)
    assert list(cy) == kat["cylindrical_x"] == [0.0, 0.5]
    u = (C.c_uint32 * 16)()
    L.orc_rng_u32(1, 0, 16, u, 0)
    assert list(u) == kat["pcg_seed1_stream0"]
    L.orc_rng_u32(42, 0x4000000000000001, 16, u, 0)
    assert list(u) == kat["pcg_seed42_init"]
    for p, x in zip((1e-10, 0.01, 0.3, 0.5, 0.9, 0.99999), kat["normal_quantile"]):
        assert L.orc_normal_quantile(p) == x


def test_philox_known_answers(oracle_lib):
    """Philox4x32-10 known-answer vectors (Salmon et al., SC'11, Random123 kat set)."""
    L = oracle_lib.lib
    cases = [
        ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
        ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
        ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
         (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
    ]
    for ctr, key, want in cases:
        out = (C.c_uint32 * 4)()
        L.orc_philox_block((C.c_uint32 * 4)(*ctr), (C.c_uint32 * 2)(*key), out)
        assert tuple(out) == want


def test_truncated_normal_properties(oracle_lib):
    """sampler within [-pi, pi], P(|theta| <= 1) at sigma = 1,
    pdf integrates to 1 for sigma in {1e-3, 0.1, 1, 10}."""
    L = oracle_lib.lib
    n = 200000
    out = np.zeros(n)
    L.orc_angular_sample(1.0, 3, 9, n, out.ctypes.data_as(C.POINTER(C.c_double)), 0)
    assert np.all(np.abs(out) <= np.pi)
    p = np.mean(np.abs(out) <= 1.0)
    assert abs(p - 0.68382) < 4 * np.sqrt(0.68382 * 0.31618 / n)
    assert abs(out.mean()) < 0.01
    for sigma in (1e-3, 0.1, 1.0, 10.0):
        th = np.linspace(-np.pi, np.pi, 400001)
        pdf = np.zeros_like(th)
        pv, sa = C.c_double(), C.c_double()
        sel = th[:: 1] if sigma >= 0.1 else np.linspace(-20 * sigma, 20 * sigma, 400001)
        vals = []
        for t in sel[::50]:
            L.orc_angular_pdf(sigma, t, C.byref(pv), C.byref(sa))
            vals.append(pv.value)
        vals = np.array(vals)
        integral = np.trapezoid(vals, sel[::50])
        assert integral == pytest.approx(1.0, abs=2e-5), sigma
        del pdf


def test_rrmse_formula_matches_reference(ref_lib):
    """The metrics rRMSE (error_report, core/diagnostics.cpp:11-38, luminance,
    eps 1e-2): numpy checker == the reference's function; and the reference's
    last metrics row with RenderConfig::reference set equals error_report of
    its final image."""
    from oracle.abi import OracleConfig, np_error_report, ref_error_report, ref_set_reference
    from paper_2402_08273_b200 import scenes
    rng = np.random.default_rng(3)
    a = rng.random((16, 24, 3), dtype=np.float32) * 2
    b = rng.random((16, 24, 3), dtype=np.float32)
    assert abs(np_error_report(a, b) - ref_error_report(ref_lib, a, b)) <= 1e-14 * ref_error_report(ref_lib, a, b)
    cfg = OracleConfig(strategy="fixed", perturbation="lens", chains=8, mutations=8 * 40, width=24, height=16,
                       max_vertices=9, b_samples=4096, seed=5, metrics_interval=8 * 10)
    ref_set_reference(ref_lib, b)
    try:
        o = ref_lib.render(scenes.cornell_box(), cfg)
    finally:
        ref_set_reference(ref_lib, None)
    rr = o.metrics[:, 2]
    assert len(rr) == 4 and np.all(np.isfinite(rr))
    assert rr[-1] == ref_error_report(ref_lib, o.image, b)


def test_pfm_io_matches_reference(ref_lib, tmp_path):
    """paper_2402_08273_b200.image_io mirrors write_pfm / read_pfm
    (core/image_io.cpp:15-56): byte-identical files, each reads the other's,
    big-endian input, and the reference's error messages."""
    import ctypes as C
    from paper_2402_08273_b200.image_io import read_pfm, write_pfm
    L = ref_lib.lib
    L.ref_write_pfm.argtypes = [C.POINTER(C.c_float), C.c_int, C.c_int, C.c_char_p]
    L.ref_read_pfm.argtypes = [C.c_char_p, C.POINTER(C.c_float), C.c_int, C.POINTER(C.c_int),
                               C.POINTER(C.c_int), C.c_char_p, C.c_int]
    img = np.random.default_rng(1).random((7, 5, 3), dtype=np.float32)
    a, b = str(tmp_path / "a.pfm"), str(tmp_path / "b.pfm")
    write_pfm(img, a)
    assert L.ref_write_pfm(np.ascontiguousarray(img).ctypes.data_as(C.POINTER(C.c_float)), 5, 7, b.encode()) == 0
    assert open(a, "rb").read() == open(b, "rb").read()
    out = np.zeros_like(img)
    w, h = C.c_int(), C.c_int()
    err = C.create_string_buffer(256)
    assert L.ref_read_pfm(a.encode(), out.ctypes.data_as(C.POINTER(C.c_float)), 35, C.byref(w), C.byref(h), err,
                          256) == 0
    assert np.array_equal(out, img) and np.array_equal(read_pfm(b), img)
    big = str(tmp_path / "big.pfm")
    with open(big, "wb") as f:
        f.write(b"PF\n5 7\n1.0\n" + img[::-1].astype(">f4").tobytes())
    assert np.array_equal(read_pfm(big), img)
    for content, msg in ((b"P6\n1 1\n-1\n", "is not a color PFM file"), (b"PF\n0 1\n-1\n", "malformed PFM header"),
                         (b"PF\n2 2\n-1\n" + b"\0" * 8, "truncated PFM data")):
        bad = str(tmp_path / "bad.pfm")
        open(bad, "wb").write(content)
        with pytest.raises(RuntimeError, match=msg):
            read_pfm(bad)
        assert L.ref_read_pfm(bad.encode(), out.ctypes.data_as(C.POINTER(C.c_float)), 35, C.byref(w), C.byref(h),
                              err, 256) == 1 and msg in err.value.decode()

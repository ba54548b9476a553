"""The C-ABI boundary (include/ramlt_gpu.h) without a GPU: the library loads,
exports exactly the declared entry points, mirrors the reference's scene
grammar and error messages, and the product path fails loudly (no CPU
fallback) when no device is present."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT, has_gpu

HEADERS = [os.path.join(ROOT, "include", h) for h in ("ramlt_gpu.h", "ramlt_mix.h")]


def declared_symbols():
    text = "".join(open(h).read() for h in HEADERS)
    return sorted(set(re.findall(r"RAMLT_API[^;(]*?\b(ramlt_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2402_08273_b200 import _capi
    lib = _capi.load()
    names = declared_symbols()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_capi.SIGNATURES), set(names) ^ set(_capi.SIGNATURES)
    out = os.popen(f"nm -D --defined-only {_capi.LIB_PATH}").read()
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert {s for s in exported if s.startswith("ramlt_")} == set(names)
    assert lib.ramlt_gpu_abi_version() == 2


def test_struct_layouts_match_header():
    """ctypes mirrors of the descriptors have the C sizes (compiled probe)."""
    import subprocess
    import tempfile
    from paper_2402_08273_b200 import _capi
    src = '#include "ramlt_gpu.h"\n#include <stdio.h>\nint main(){printf("%zu %zu %zu %zu %zu %zu %zu",' \
          'sizeof(ramlt_render_desc),sizeof(ramlt_stats),sizeof(ramlt_scene_desc),sizeof(ramlt_material),' \
          'sizeof(ramlt_triangle),sizeof(ramlt_sphere),sizeof(ramlt_trace_row));}'
    with tempfile.TemporaryDirectory() as d:
        open(os.path.join(d, "p.c"), "w").write(src)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), os.path.join(d, "p.c"), "-o",
                        os.path.join(d, "p")], check=True)
        sizes = [int(x) for x in subprocess.run([os.path.join(d, "p")], capture_output=True,
                                                 text=True).stdout.split()]
    mine = [C.sizeof(t) for t in (_capi.ramlt_render_desc, _capi.ramlt_stats, _capi.ramlt_scene_desc,
                                  _capi.ramlt_material, _capi.ramlt_triangle, _capi.ramlt_sphere,
                                  _capi.ramlt_trace_row)]
    assert sizes == mine
    src = '#include "ramlt_mix.h"\n#include <stdio.h>\nint main(){printf("%zu %zu %zu",' \
          'sizeof(ramlt_mix_target),sizeof(ramlt_mix_desc),sizeof(ramlt_mix_stats));}'
    with tempfile.TemporaryDirectory() as d:
        open(os.path.join(d, "p.c"), "w").write(src)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), os.path.join(d, "p.c"), "-o",
                        os.path.join(d, "p")], check=True)
        sizes = [int(x) for x in subprocess.run([os.path.join(d, "p")], capture_output=True,
                                                 text=True).stdout.split()]
    assert sizes == [C.sizeof(t) for t in (_capi.ramlt_mix_target, _capi.ramlt_mix_desc,
                                           _capi.ramlt_mix_stats)]


def test_target_harness_validation_before_device():
    """ramlt_mix_create validates the target (Cholesky) and the config before
    touching a device: std::invalid_argument / logic_error as the reference's
    sampling.cpp:63 / RAMLT_CHECK would raise."""
    from paper_2402_08273_b200 import LogicError
    from paper_2402_08273_b200.mix import MixConfig, MixEngine, MixTarget
    t = MixTarget.config2(0)
    bad = MixTarget(t.weights, t.means, t.covariances.copy())
    bad.covariances[2, 0, 0] = -1.0
    bad.covariances[2] = 0.5 * (bad.covariances[2] + bad.covariances[2].T)
    with pytest.raises(ValueError, match="positive definite"):
        MixEngine(bad, MixConfig())
    with pytest.raises(ValueError, match="weights"):
        MixEngine(MixTarget(-t.weights, t.means, t.covariances), MixConfig())
    with pytest.raises(LogicError):
        MixEngine(t, MixConfig(chains=0))
    with pytest.raises(LogicError):
        MixEngine(t, MixConfig(strategy="ra-grid", grid_n=0))


def test_default_desc_matches_reference_defaults():
    from paper_2402_08273_b200 import RenderConfig, _capi
    d = _capi.ramlt_render_desc()
    _capi.load().ramlt_gpu_default_desc(C.byref(d))
    # RenderConfig / AdaptationConfig defaults (core/driver.hpp:19-39, adaptation.hpp:14-22)
    assert (d.strategy, d.perturbation, d.mutations, d.chains) == (3, 0, 1_000_000, 1)
    assert (d.batch_size, d.gamma_max, d.gamma_scale, d.target_acceptance) == (10, 1.0, 5.0, 0.5)
    assert (d.lambda_init, d.lambda_min, d.sigma2_ratio) == (1.0, -30.0, 1.0)
    assert (d.n_top, d.n_bottom, d.m_split, d.m_refine) == (20, 50, 5000, 10_000_000)
    assert (d.b_samples, d.seed, d.width, d.height, d.max_vertices) == (1_000_000, 1, 256, 256, 20)
    assert d.metrics_interval == 1_000_000
    c = RenderConfig()
    assert (c.strategy, c.mutations, c.m_refine, c.max_vertices) == ("ra-quadtree", 1_000_000, 10_000_000, 20)


BAD_SCENES = [
    ("camera 0 0 0 0 0 1 0 1 0 45\nmaterial a diffuse 2 0 0\n", "<s>:2: albedo components must be in [0,1]"),
    ("camera 0 0 0 0 0 1 0 1 0 45\nmaterial a glass 1\n", "<s>:2: unknown material kind 'glass'"),
    ("camera 0 0 0 0 0 1 0 1 0 45\ntri 0 0 0 1 0 0 0 1 0 x\n", "<s>:2: unknown material 'x'"),
    ("camera 0 0 0 0 0 1 0 1 0 190\n", "<s>:1: camera: fov must be in (0, 180) degrees"),
    ("camera 0 0 0 0 0 1 0 0 1 45\n", "<s>:1: camera: up vector is parallel to the view direction"),
    ("camera 0 0 0 0 0 1 0 1 0 45\nmaterial m diffuse 1 1 1\nsphere 0 0 3 1 m\n", "<s>: scene has no emitter"),
    ("material m diffuse 1 1 1\n", "<s>: scene has no camera"),
    ("camera 0 0 0 0 0 1 0 1 0 45\nmaterial m diffuse 1 1 1\nsphere 0 0 3 -1 m\n", "<s>:3: sphere radius must be > 0"),
    ("camera 0 0 0 0 0 1 0 1 0 45\nmaterial m diffuse 1 1 1\nsphere 0 0 3 1 m\nemitter 4 1 1 1\n",
     "<s>:4: emitter geometry index out of range"),
    ("camera 0 0 0 0 0 1 0 1 0 45\nmaterial m diffuse 1 1 1\nsphere 0 0 3 1 m\nemitter 0 -1 1 1\n",
     "<s>:4: emitted radiance must be non-negative"),
    ("camera 0 0 0 0 0 1 0 1 0 45\nbogus 1\n", "<s>:2: unknown record 'bogus'"),
    ("camera 0 0 0 0 0 1 0 1\n", "<s>:1: malformed 'camera' record"),
    ("camera 0 0 0 0 0 1 0 1 0 45\nmaterial m dielectric 0.9 1 1 1\n", "<s>:2: dielectric ior must be > 1"),
    ("camera 0 0 0 0 0 1 0 1 0 45\nmaterial m diffuse 1 1 1\nmaterial m diffuse 1 1 1\n",
     "<s>:3: duplicate material 'm'"),
]


@pytest.mark.parametrize("text,msg", BAD_SCENES)
def test_scene_parse_errors_mirror_reference(text, msg):
    from paper_2402_08273_b200 import parse_scene
    with pytest.raises(RuntimeError) as e:
        parse_scene(text, "<s>")
    assert str(e.value) == msg


@pytest.mark.parametrize("text,msg", BAD_SCENES)
def test_scene_parse_errors_equal_reference_text(ref_lib, text, msg):
    err = C.create_string_buffer(512)
    counts = (C.c_int * 4)()
    rc = ref_lib.lib.ref_parse(text.encode(), counts, err, 512)
    assert rc == 1
    assert err.value.decode().replace("<scene>", "<s>") == msg


def test_scene_counts_match_reference(ref_lib):
    from paper_2402_08273_b200 import parse_scene, scenes
    for name, fn in scenes.SCENES.items():
        text = fn()
        counts = (C.c_int * 4)()
        err = C.create_string_buffer(256)
        assert ref_lib.lib.ref_parse(text.encode(), counts, err, 256) == 0
        assert tuple(counts) == parse_scene(text).counts, name


@pytest.mark.skipif(has_gpu(), reason="checks the no-device behaviour")
def test_engine_fails_loudly_without_gpu():
    from paper_2402_08273_b200 import CudaError, Engine, RenderConfig, scenes
    with pytest.raises(CudaError):
        Engine(scenes.cornell_box(), RenderConfig(chains=4))


def test_invalid_config_errors_before_device():
    """RAMLT_CHECK-style validation (driver.cpp:178-180) happens before any
    device work and raises the reference's logic_error."""
    from paper_2402_08273_b200 import Engine, LogicError, RenderConfig, scenes
    for bad in (dict(chains=0), dict(width=0), dict(max_vertices=1)):
        with pytest.raises(LogicError):
            Engine(scenes.cornell_box(), RenderConfig(**bad))
    with pytest.raises(ValueError):
        Engine(scenes.cornell_box(), RenderConfig(max_vertices=40))


def _parsed_prims(text):
    from paper_2402_08273_b200 import parse_scene
    sc = parse_scene(text, "<s>")
    d = sc.desc
    tris = [(tuple(t.a) + tuple(t.b) + tuple(t.c), t.material, t.emitter)
            for t in (d.triangles[i] for i in range(d.n_triangles))]
    sphs = [(tuple(s.center) + (s.radius,), s.material, s.emitter)
            for s in (d.spheres[i] for i in range(d.n_spheres))]
    return tris, sphs


def _py_prims(text):
    """Independent parse of the geometry records: Python's float() is
    correctly rounded, like the reference stream's strtod."""
    mats, tris, sphs, order = {}, [], [], []
    for line in text.split("\n"):
        tok = line.split()
        if not tok or tok[0].startswith("#"):
            continue
        if tok[0] == "material":
            mats[tok[1]] = len(mats)
        elif tok[0] == "tri":
            order.append(("t", len(tris)))
            tris.append([tuple(float(x) for x in tok[1:10]), mats[tok[10]], -1])
        elif tok[0] == "sphere":
            order.append(("s", len(sphs)))
            sphs.append([tuple(float(x) for x in tok[1:5]), mats[tok[5]], -1])
        elif tok[0] == "emitter":
            kind, i = order[int(tok[1])]
            (tris if kind == "t" else sphs)[i][2] = sum(1 for t in tris if t[2] >= 0) + \
                sum(1 for s in sphs if s[2] >= 0)
    return [tuple(t) for t in tris], [tuple(s) for s in sphs]


def test_scene_parse_values_bit_exact():
    """The from_chars fast path and the stream path parse every coordinate to
    the correctly rounded double (bit-exact with the reference's strtod)."""
    from paper_2402_08273_b200 import scenes
    odd = ("camera 0 0 -3 0 0 0 0 1 0 45\nmaterial m diffuse 0.5 0.5 0.5\n"
           "tri +1 .5 1. 1E3 -0 0.1000000000000000055511151231257827 1e-5 2.5e+2 7 m\n"
           "tri 0.3 0.30000000000000004 1e-320 3 4 5 6 7 8   m   trailing tokens\n"
           "  \t sphere 0 0 3 1 m\r\n# comment\n\nsphere +0 -0 3.0 .25 m\nemitter 3 1 1 1\n")
    texts = [fn() for fn in (scenes.cornell_box, scenes.caustic_box, scenes.mirror_box)]
    texts += [scenes.cluster_room(n_tris=2000), odd]
    for text in texts:
        tris, sphs = _parsed_prims(text)
        ptris, psphs = _py_prims(text)
        assert len(tris) == len(ptris) and len(sphs) == len(psphs)
        for got, want in zip(tris + sphs, ptris + psphs):
            assert got[0] == want[0] and got[1] == want[1]


@pytest.mark.parametrize("rec", ["tri 0 0 0 1 0 0 0 1 inf m", "tri 0 0 0 1 0 0 0 1 nan m",
                                 "tri 0 0 0 1 0 0 0 1 0x1p1 m", "tri 0 0 0 1 0 0 0 1 1e999 m",
                                 "tri 0 0 0 1 0 0 0 1 m", "sphere 0 0 1e999 1 m", "tri 0 0 0 1 0 0 0 1 2,5 m"])
def test_scene_parse_odd_numbers_match_reference(ref_lib, rec):
    """Tokens the fast path does not take fall back to the stream path: same
    result (accepted or the same error) as the reference parser."""
    from paper_2402_08273_b200 import parse_scene
    text = f"camera 0 0 -3 0 0 0 0 1 0 45\nmaterial m diffuse 0.5 0.5 0.5\nsphere 0 0 3 1 m\nemitter 0 1 1 1\n{rec}\n"
    err = C.create_string_buffer(512)
    counts = (C.c_int * 4)()
    rc = ref_lib.lib.ref_parse(text.encode(), counts, err, 512)
    if rc == 0:
        assert parse_scene(text, "<s>").counts == tuple(counts)
    else:
        with pytest.raises(RuntimeError) as e:
            parse_scene(text, "<s>")
        assert str(e.value) == err.value.decode().replace("<scene>", "<s>")

"""Synthetic scene generators for the BASELINE.json configs, emitted as the
reference's line-oriented ``.scn`` grammar (parser at
core/scene.cpp:114-234), so the identical text feeds the GPU engine and the CPU
checkers.

The paper's scenes (Fireplace Room, Necklace, ...) are not available here;
these seeded stand-ins follow the shapes and sizes named in BASELINE.json and
SURVEY.md §8(d):

* ``cornell_box``   -- C1: unit room with an open front, 5 diffuse walls
  (2 triangles each), 2 axis-aligned diffuse boxes (12 triangles each) and one
  quad area light (2 triangles, radiance 17 x 12 x 4, facing -y just below the
  ceiling): 36 triangles.
* ``caustic_box``   -- C3: the same box plus a dielectric sphere (ior 1.5,
  transmittance 1, radius 0.25 box widths) resting on the short box, with the
  light shrunk to 1 % of the ceiling area.
* ``cluster_room``  -- C4/C5: closed room (12 triangles), 4 ceiling quad lights
  (8 triangles) and ``n_tris`` small random triangles in 64 seeded clusters
  (edge lengths U(0.001, 0.02)); camera inside the room.
"""
from __future__ import annotations

import numpy as np

# Diffuse albedos chosen for the stand-in (recorded here).
WHITE = (0.73, 0.73, 0.73)
RED = (0.65, 0.05, 0.05)
GREEN = (0.12, 0.45, 0.15)
LIGHT_RADIANCE = (17.0, 12.0, 4.0)


class _SceneText:
    def __init__(self) -> None:
        self.lines: list[str] = []
        self.geometry = 0

    def camera(self, pos, look, up, fov):
        self.lines.append("camera %r %r %r  %r %r %r  %r %r %r  %r" % (*pos, *look, *up, fov))

    def material(self, name, kind, *vals):
        self.lines.append("material %s %s %s" % (name, kind, " ".join(repr(float(v)) for v in vals)))

    def tri(self, a, b, c, mat) -> int:
        self.lines.append(
            "tri %r %r %r  %r %r %r  %r %r %r %s" % (*map(float, a), *map(float, b), *map(float, c), mat))
        self.geometry += 1
        return self.geometry - 1

    def quad(self, p0, p1, p2, p3, mat) -> tuple[int, int]:
        return self.tri(p0, p1, p2, mat), self.tri(p0, p2, p3, mat)

    def sphere(self, c, r, mat) -> int:
        self.lines.append("sphere %r %r %r %r %s" % (*map(float, c), float(r), mat))
        self.geometry += 1
        return self.geometry - 1

    def emitter(self, index, radiance):
        self.lines.append("emitter %d %r %r %r" % (index, *map(float, radiance)))

    def box(self, lo, hi, mat):
        x0, y0, z0 = lo
        x1, y1, z1 = hi
        self.quad((x0, y0, z0), (x1, y0, z0), (x1, y0, z1), (x0, y0, z1), mat)  # bottom
        self.quad((x0, y1, z0), (x0, y1, z1), (x1, y1, z1), (x1, y1, z0), mat)  # top
        self.quad((x0, y0, z0), (x0, y1, z0), (x1, y1, z0), (x1, y0, z0), mat)  # front
        self.quad((x0, y0, z1), (x1, y0, z1), (x1, y1, z1), (x0, y1, z1), mat)  # back
        self.quad((x0, y0, z0), (x0, y0, z1), (x0, y1, z1), (x0, y1, z0), mat)  # left
        self.quad((x1, y0, z0), (x1, y1, z0), (x1, y1, z1), (x1, y0, z1), mat)  # right

    def ceiling_light(self, cx, cz, half, y, radiance, mat="light"):
        # Winding chosen so normalize(cross(b-a, c-a)) = -y: emission is
        # one-sided from the front face (core/path.cpp:31-38).
        a = (cx - half, y, cz - half)
        b = (cx + half, y, cz - half)
        c = (cx + half, y, cz + half)
        d = (cx - half, y, cz + half)
        t0 = self.tri(a, b, c, mat)
        t1 = self.tri(a, c, d, mat)
        self.emitter(t0, radiance)
        self.emitter(t1, radiance)

    def text(self) -> str:
        return "\n".join(self.lines) + "\n"


def _open_box_walls(s: _SceneText) -> None:
    s.quad((0, 0, 0), (1, 0, 0), (1, 0, 1), (0, 0, 1), "white")  # floor
    s.quad((0, 1, 0), (0, 1, 1), (1, 1, 1), (1, 1, 0), "white")  # ceiling
    s.quad((0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1), "white")  # back
    s.quad((0, 0, 0), (0, 0, 1), (0, 1, 1), (0, 1, 0), "red")    # left
    s.quad((1, 0, 0), (1, 1, 0), (1, 1, 1), (1, 0, 1), "green")  # right


def cornell_box(light_half: float = 0.12) -> str:
    """C1: 36 triangles (BASELINE.json configs[0])."""
    s = _SceneText()
    s.lines.append("# C1 stand-in: Cornell-style open box, 36 triangles")
    s.camera((0.5, 0.5, -1.0), (0.5, 0.5, 0.5), (0.0, 1.0, 0.0), 45.0)
    s.material("white", "diffuse", *WHITE)
    s.material("red", "diffuse", *RED)
    s.material("green", "diffuse", *GREEN)
    s.material("light", "diffuse", 0.0, 0.0, 0.0)
    _open_box_walls(s)
    s.box((0.53, 0.0, 0.15), (0.83, 0.30, 0.45), "white")  # short box
    s.box((0.17, 0.0, 0.50), (0.47, 0.60, 0.80), "white")  # tall box
    s.ceiling_light(0.5, 0.5, light_half, 0.999, LIGHT_RADIANCE)
    return s.text()


def caustic_box() -> str:
    """C3: C1 + glass sphere (ior 1.5, r = 0.25) + light at 1 % of the ceiling."""
    s = _SceneText()
    s.lines.append("# C3 stand-in: Cornell box + dielectric sphere + small light")
    s.camera((0.5, 0.5, -1.0), (0.5, 0.5, 0.5), (0.0, 1.0, 0.0), 45.0)
    s.material("white", "diffuse", *WHITE)
    s.material("red", "diffuse", *RED)
    s.material("green", "diffuse", *GREEN)
    s.material("light", "diffuse", 0.0, 0.0, 0.0)
    s.material("glass", "dielectric", 1.5, 1.0, 1.0, 1.0)
    _open_box_walls(s)
    s.box((0.53, 0.0, 0.15), (0.83, 0.30, 0.45), "white")
    s.box((0.17, 0.0, 0.50), (0.47, 0.60, 0.80), "white")
    s.sphere((0.68, 0.55, 0.30), 0.25, "glass")
    s.ceiling_light(0.5, 0.5, 0.05, 0.999, LIGHT_RADIANCE)  # 0.1 x 0.1 = 1 %
    return s.text()


def mirror_box() -> str:
    """Small mixed-material scene (mirror + glossy + dielectric) for parity tests."""
    s = _SceneText()
    s.lines.append("# mixed-material parity scene")
    s.camera((0.5, 0.5, -1.0), (0.5, 0.5, 0.5), (0.0, 1.0, 0.0), 45.0)
    s.material("white", "diffuse", *WHITE)
    s.material("red", "diffuse", *RED)
    s.material("green", "glossy", 0.2, 0.6, 0.2, 20.0)
    s.material("light", "diffuse", 0.0, 0.0, 0.0)
    s.material("mirror", "mirror", 0.95, 0.95, 0.95)
    s.material("glass", "dielectric", 1.5, 1.0, 1.0, 1.0)
    _open_box_walls(s)
    s.box((0.17, 0.0, 0.50), (0.47, 0.60, 0.80), "mirror")
    s.sphere((0.68, 0.2, 0.35), 0.2, "glass")
    s.ceiling_light(0.5, 0.5, 0.15, 0.999, LIGHT_RADIANCE)
    return s.text()


def cluster_room(n_tris: int = 1 << 20, clusters: int = 64, seed: int = 7) -> str:
    """C4/C5: closed room + 4 ceiling lights + n_tris random triangles in clusters."""
    rng = np.random.default_rng(seed)
    s = _SceneText()
    s.lines.append("# C4 stand-in: closed room, 4 lights, %d clustered triangles" % n_tris)
    s.camera((0.5, 0.45, 0.02), (0.5, 0.4, 1.0), (0.0, 1.0, 0.0), 60.0)
    s.material("white", "diffuse", *WHITE)
    s.material("red", "diffuse", *RED)
    s.material("green", "diffuse", *GREEN)
    s.material("light", "diffuse", 0.0, 0.0, 0.0)
    s.material("clay", "diffuse", 0.6, 0.55, 0.5)
    _open_box_walls(s)
    s.quad((0, 0, 0), (0, 1, 0), (1, 1, 0), (1, 0, 0), "white")  # front wall closes the room
    for cx, cz in ((0.3, 0.3), (0.7, 0.3), (0.3, 0.7), (0.7, 0.7)):
        s.ceiling_light(cx, cz, 0.06, 0.999, (6.0, 5.0, 3.0))
    centres = rng.uniform(0.15, 0.85, size=(clusters, 3))
    centres[:, 1] = rng.uniform(0.1, 0.6, size=clusters)
    per = np.full(clusters, n_tris // clusters)
    per[: n_tris - per.sum()] += 1
    out = []
    for c, m in zip(centres, per):
        spread = rng.uniform(0.02, 0.08)
        p0 = c + rng.normal(0.0, spread, size=(m, 3))
        p0 = np.clip(p0, 0.01, 0.99)
        edge = rng.uniform(0.001, 0.02, size=(m, 1))
        d1 = rng.normal(size=(m, 3))
        d1 /= np.linalg.norm(d1, axis=1, keepdims=True)
        d2 = rng.normal(size=(m, 3))
        d2 /= np.linalg.norm(d2, axis=1, keepdims=True)
        p1 = p0 + edge * d1
        p2 = p0 + edge * d2
        out.append(np.concatenate([p0, p1, p2], axis=1))
    tris = np.concatenate(out, axis=0)
    body = "\n".join("tri " + " ".join("%.7f" % v for v in row) + " clay" for row in tris)
    return s.text() + body + "\n"


SCENES = {
    "cornell": cornell_box,
    "caustic": caustic_box,
    "mirror": mirror_box,
    "clusters": cluster_room,
}

"""Canonical synthetic workloads of BASELINE.json.

All of them are expressible with the reference's scene vocabulary, so the
same scene drives the CUDA path and the reference/oracle CPU path:

  C1  homogeneous isotropic cube (albedo 0.9), one area light, 64x64, 4 spp,
      max_depth 16, 10 iterations                     (runs on the CPU reference)
  C2  256^3 fbm cloud, HG g=0.8, albedo 0.99, sun + area light, 512x512, 8 spp
  C3  dense forward-scattering homogeneous block (g=0.9, albedo 0.995),
      512x512, 16 spp (the dielectric boundary is not expressible: omitted)
  C4  512^3 fbm smoke, g=0.3, five-quad sky dome, 1024x1024, 16 spp, 16 iterations
  C5  the C2 scene at 2048x2048, 64 spp (~1B vertices, multi-GPU)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2404_11894_b200.scenecore.types import Camera, Emitter, Medium, Scene, Surface

CAMERA_ORIGIN = (0.0, 0.4, -4.2)
LIGHT_QUAD = (-0.6, 1.6, -0.6, 1.2, 0.0, 0.0, 0.0, 0.0, 1.2)


def fbm_density(n: int, seed: int, squash: float) -> np.ndarray:
    """Procedural cloud: a squashed sphere falloff plus 5 octaves of separable
    sine noise, clipped at 0 and normalised to max 1, float32 (z, y, x)."""
    ax = np.linspace(-1.0, 1.0, n, dtype=np.float32)
    rng = np.random.default_rng(seed)
    octaves = []
    for o in range(5):
        f = np.float32(2.0 ** (o + 1))
        phase = (rng.random(3) * 2.0 * np.pi).astype(np.float32)
        amp = np.float32(0.5 ** o)
        octaves.append((amp,
                        np.sin(f * np.float32(3.1) * ax + phase[0]),
                        np.sin(f * np.float32(2.7) * ax + phase[1]),
                        np.sin(f * np.float32(3.3) * ax + phase[2])))
    out = np.empty((n, n, n), dtype=np.float32)
    x2 = (ax * ax)[None, None, :]
    y2 = (np.float32(squash) * ax * ax)[None, :, None]
    slab = max(1, (1 << 24) // (n * n))
    for z0 in range(0, n, slab):
        z = ax[z0:z0 + slab]
        r = np.sqrt(x2 + y2 + (z * z)[:, None, None])
        acc = np.zeros_like(r)
        for amp, sx, sy, sz in octaves:
            acc += amp * sz[z0:z0 + slab, None, None] * sy[None, :, None] * sx[None, None, :]
        np.maximum(np.float32(1.0) - r + np.float32(0.35) * acc, np.float32(0.0),
                   out=out[z0:z0 + slab])
    out /= out.max()
    return out


def _area_light(value=(10.0, 10.0, 10.0), quad=LIGHT_QUAD):
    return Surface("quad", quad, "emitter", emitter_index=0), Emitter("area", value)


def _camera(fov, res):
    return Camera(CAMERA_ORIGIN, (0.0, 0.0, 0.0), float(fov), (int(res[0]), int(res[1])))


def scene_c1(res=(64, 64), floor: bool = False) -> Scene:
    quad, light = _area_light()
    med = Medium("homogeneous", (2.0, 2.0, 2.0), (1.8, 1.8, 1.8), 0.0, (-1, -1, -1, 1, 1, 1),
                 name="fog")
    surfaces = [quad]
    if floor:  # a Lambertian floor adds a surface class (two compatibility classes)
        surfaces.append(Surface("quad", (-3.0, -1.2, 3.0, 6.0, 0.0, 0.0, 0.0, 0.0, -6.0),
                                "lambertian", albedo=(0.6, 0.6, 0.6)))
    return Scene(_camera(32.0, res), [med], surfaces, [light])


def scene_mixed(res=(12, 12)) -> Scene:
    """Test scene covering what the configs do not: a chromatic, anisotropic
    homogeneous medium, sphere and box surfaces (Lambertian and black), a
    floor, and a point light beside the area light (delta and non-delta
    emitters, several surface compatibility classes)."""
    quad, light = _area_light()
    med = Medium("homogeneous", (2.0, 1.5, 1.0), (1.6, 1.2, 0.7), 0.5, (-1, -1, -1, 1, 1, 1),
                 name="haze")
    surfaces = [
        quad,
        Surface("sphere", (0.35, -0.3, 0.2, 0.35), "lambertian", albedo=(0.8, 0.5, 0.3)),
        Surface("box", (-0.8, -0.9, -0.3, -0.4, -0.5, 0.3), "lambertian", albedo=(0.3, 0.6, 0.9)),
        Surface("box", (0.3, 0.4, -0.6, 0.6, 0.7, -0.2), "black"),
        Surface("quad", (-3.0, -1.2, 3.0, 6.0, 0.0, 0.0, 0.0, 0.0, -6.0), "lambertian",
                albedo=(0.6, 0.6, 0.6)),
    ]
    point = Emitter("point", (3.0, 2.5, 2.0), position=(-0.5, 0.8, -1.5))
    return Scene(_camera(32.0, res), [med], surfaces, [light, point])


def scene_c2(res=(512, 512), grid_n: int = 256) -> Scene:
    quad, light = _area_light()
    sun = Emitter("directional", (3.0, 2.9, 2.6), direction=(0.3, -1.0, 0.2))
    dens = fbm_density(grid_n, seed=2, squash=1.0)
    med = Medium("grid", (16.0, 16.0, 16.0), (15.84, 15.84, 15.84), 0.8, (-1, -1, -1, 1, 1, 1),
                 name="cloud", density=dens)
    return Scene(_camera(28.0, res), [med], [quad], [light, sun])


def scene_c3(res=(512, 512)) -> Scene:
    quad, light = _area_light()
    med = Medium("homogeneous", (20.0, 20.0, 20.0), (19.9, 19.9, 19.9), 0.9,
                 (-0.7, -0.7, -0.7, 0.7, 0.7, 0.7), name="dense")
    return Scene(_camera(32.0, res), [med], [quad], [light])


def scene_fogbox(res=(128, 128), half: float = 0.5) -> Scene:
    """SPEC.md acceptance scene FogBox: homogeneous cube, sigma_s 1.8,
    sigma_a 0.2, HG g = 0.5, one area light.  The SPEC leaves the cube's size
    open: the default is the unit cube (optical depth 2 across); at half = 1
    (optical depth 4) the reference's own fixed-point iteration diverges from
    128x128 at 1 spp (tests/test_gpu_acceptance.py checks the device diverges
    with it)."""
    quad, light = _area_light()
    h = float(half)
    med = Medium("homogeneous", (2.0, 2.0, 2.0), (1.8, 1.8, 1.8), 0.5, (-h, -h, -h, h, h, h),
                 name="fogbox")
    return Scene(_camera(32.0, res), [med], [quad], [light])


def scene_gridpuff(res=(256, 256), grid_n: int = 32, half: float = 0.5) -> Scene:
    """SPEC.md acceptance scene GridPuff: FogBox as a constant-density grid
    (delta / ratio tracking instead of the closed forms)."""
    quad, light = _area_light()
    dens = np.ones((grid_n, grid_n, grid_n), dtype=np.float32)
    h = float(half)
    med = Medium("grid", (2.0, 2.0, 2.0), (1.8, 1.8, 1.8), 0.5, (-h, -h, -h, h, h, h),
                 name="gridpuff", density=dens)
    return Scene(_camera(32.0, res), [med], [quad], [light])


DOME = [  # (origin, edge_u, edge_v) of the five inward-facing sky quads
    ((-6.0, 6.0, -6.0), (12.0, 0.0, 0.0), (0.0, 0.0, 12.0)),
    ((-6.0, -6.0, 6.0), (0.0, 12.0, 0.0), (12.0, 0.0, 0.0)),
    ((-6.0, -6.0, -6.0), (12.0, 0.0, 0.0), (0.0, 12.0, 0.0)),
    ((6.0, -6.0, -6.0), (0.0, 0.0, 12.0), (0.0, 12.0, 0.0)),
    ((-6.0, -6.0, -6.0), (0.0, 12.0, 0.0), (0.0, 0.0, 12.0)),
]


def scene_c4(res=(1024, 1024), grid_n: int = 512) -> Scene:
    surfaces, emitters = [], []
    for i, (o, u, v) in enumerate(DOME):
        surfaces.append(Surface("quad", o + u + v, "emitter", emitter_index=i))
        emitters.append(Emitter("area", (0.6, 0.75, 1.0)))
    dens = fbm_density(grid_n, seed=4, squash=0.8)
    med = Medium("grid", (16.0, 16.0, 16.0), (15.84, 15.84, 15.84), 0.3, (-1, -1, -1, 1, 1, 1),
                 name="smoke", density=dens)
    return Scene(_camera(28.0, res), [med], surfaces, emitters)


@dataclass(frozen=True)
class Workload:
    name: str
    res: tuple
    spp: int
    max_depth: int
    iterations: int
    grid_n: int = 0

    def scene(self, res=None) -> Scene:
        res = res or self.res
        if self.name == "C1":
            return scene_c1(res)
        if self.name in ("C2", "C5"):
            return scene_c2(res, self.grid_n)
        if self.name == "C3":
            return scene_c3(res)
        return scene_c4(res, self.grid_n)


WORKLOADS = {
    "C1": Workload("C1", (64, 64), 4, 16, 10),
    "C2": Workload("C2", (512, 512), 8, 64, 10, 256),
    "C3": Workload("C3", (512, 512), 16, 64, 10),
    "C4": Workload("C4", (1024, 1024), 16, 64, 16, 512),
    "C5": Workload("C5", (2048, 2048), 64, 64, 10, 256),
}

"""Pack a Scene into the tracer's by-value kernel argument (vpg_scene).

Follows the reference's flattening (scenecore/flatten.py:87-195): the same
type/material/emitter codes, the quad normal and area of each area light,
directional lights stored as unit travel directions, grid volumes
concatenated as float32 (z, y, x), and the camera basis built with numpy in
the same operation order so the camera rays are bit-identical.  The density
volumes are uploaded once and cached on the Scene with the packed struct.
"""

from __future__ import annotations

import math

import numpy as np

from paper_2404_11894_b200 import _native as N
from paper_2404_11894_b200.scenecore.types import Scene, SceneError

SURF_CODES = {"sphere": 0, "box": 1, "quad": 2}
MAT_CODES = {"lambertian": 0, "black": 1, "emitter": 2}


def _unit_normal(u, v):
    """Normalised u x v, the reference's quad_normal (geometry.py:115-120)."""
    nx = u[1] * v[2] - u[2] * v[1]
    ny = u[2] * v[0] - u[0] * v[2]
    nz = u[0] * v[1] - u[1] * v[0]
    inv = 1.0 / math.sqrt(nx * nx + ny * ny + nz * nz)
    return nx * inv, ny * inv, nz * inv


def camera_basis(scene: Scene):
    """(origin, forward, right, up, tan_half) exactly as flatten.py:170-182."""
    cam = scene.camera
    origin = np.asarray(cam.origin, dtype=np.float64)
    fwd = np.asarray(cam.look_at, dtype=np.float64) - origin
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(cam.up, dtype=np.float64))
    norm = np.linalg.norm(right)
    if norm < 1e-9:
        right = np.cross(fwd, np.array([1.0, 0.0, 0.0]))
        norm = np.linalg.norm(right)
    right /= norm
    up = np.cross(right, fwd)
    return origin, fwd, right, up, float(np.tan(np.radians(cam.fov) * 0.5))


class PackedScene:
    """The vpg_scene struct plus the device tensor holding the grid volumes."""

    def __init__(self, struct: N.SceneStruct, grid_host: np.ndarray, width: int, height: int):
        self.struct = struct
        self.grid_host = grid_host
        self.width = width
        self.height = height
        self._grid_dev = None

    def device(self) -> N.SceneStruct:
        if self._grid_dev is None and self.grid_host.size:
            torch = N.require_cuda()
            self._grid_dev = torch.from_numpy(self.grid_host).to("cuda")
            self.struct.grid_data = self._grid_dev.data_ptr()
        return self.struct


def pack_scene(scene: Scene) -> PackedScene:
    cached = scene.__dict__.get("_vpg_packed")
    if cached is not None:
        return cached
    if len(scene.surfaces) > N.MAX_SURF or len(scene.emitters) > N.MAX_EMIT or \
            len(scene.media) > N.MAX_MED:
        raise SceneError(f"scene exceeds tracer limits ({N.MAX_SURF} surfaces, "
                         f"{N.MAX_EMIT} emitters, {N.MAX_MED} media)")
    st = N.SceneStruct()
    st.n_surf, st.n_emit, st.n_med = len(scene.surfaces), len(scene.emitters), len(scene.media)
    for i, s in enumerate(scene.surfaces):
        st.surf_type[i] = SURF_CODES[s.geometry]
        st.mat_type[i] = MAT_CODES[s.material]
        st.emitter_id[i] = s.emitter_index
        for a, p in enumerate(s.params):
            st.surf_params[i][a] = float(p)
        for a in range(3):
            st.albedo[i][a] = float(s.albedo[a])
    for j, e in enumerate(scene.emitters):
        for a in range(3):
            st.em_value[j][a] = float(e.value[a])
        if e.kind == "point":
            st.em_type[j] = 0
            for a in range(3):
                st.em_pos[j][a] = float(e.position[a])
        elif e.kind == "directional":
            st.em_type[j] = 2
            d = np.asarray(e.direction, dtype=np.float64)
            norm = np.linalg.norm(d)
            if norm < 1e-12:
                raise SceneError(f"directional emitter {j} has a zero direction")
            d = d / norm
            for a in range(3):
                st.em_pos[j][a] = float(d[a])
        else:
            st.em_type[j] = 1
            # the emitter's quad (types.py area_emitter_surface), found by
            # field access so any scene object with the reference's fields works
            q = next((sf.params for sf in scene.surfaces
                      if sf.material == "emitter" and sf.emitter_index == j), None)
            if q is None:
                raise SceneError(f"area emitter {j} has no surface")
            for a in range(9):
                st.em_quad[j][a] = float(q[a])
            u, v = np.asarray(q[3:6], dtype=np.float64), np.asarray(q[6:9], dtype=np.float64)
            area = float(np.linalg.norm(np.cross(u, v)))
            if area < 1e-12:
                raise SceneError(f"area emitter {j} has a degenerate quad")
            st.em_area[j] = area
            n = _unit_normal(u, v)
            for a in range(3):
                st.em_normal[j][a] = n[a]
    chunks, offset = [], 0
    for k, m in enumerate(scene.media):
        st.med_kind[k] = 0 if m.kind == "homogeneous" else 1
        for a in range(3):
            st.med_sigma_t[k][a] = float(m.sigma_t[a])
            st.med_sigma_s[k][a] = float(m.sigma_s[a])
        st.med_g[k] = float(m.phase_g)
        for a in range(6):
            st.med_bounds[k][a] = float(m.bounds[a])
        # Medium.majorant (types.py:95-101) from the fields
        top = float(max(m.sigma_t))
        st.med_majorant[k] = top if m.kind == "homogeneous" else \
            float(np.max(m.density)) * float(m.density_scale) * top
        st.med_scale[k] = float(m.density_scale)
        if m.kind == "grid":
            vol = np.ascontiguousarray(m.density, dtype=np.float32)
            nz, ny, nx = vol.shape
            st.grid_dims[k][0], st.grid_dims[k][1], st.grid_dims[k][2] = nx, ny, nz
            st.grid_offset[k] = offset
            chunks.append(vol.reshape(-1))
            offset += vol.size
    grid = np.concatenate(chunks) if chunks else np.zeros(0, dtype=np.float32)
    origin, fwd, right, up, tan_half = camera_basis(scene)
    w, h = scene.camera.resolution
    cam = list(origin) + list(fwd) + list(right) + list(up) + [tan_half, float(w), float(h)]
    for a, v in enumerate(cam):
        st.cam[a] = float(v)
    st.width, st.height = int(w), int(h)
    packed = PackedScene(st, grid, int(w), int(h))
    scene.__dict__["_vpg_packed"] = packed
    return packed

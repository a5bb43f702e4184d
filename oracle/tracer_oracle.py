"""TEST INFRASTRUCTURE ONLY — ctypes driver of oracle/tracer_oracle.c.

Flattens a scene the way the reference does (scenecore/flatten.py:87-195)
and runs the reference's two-pass capture (transport/tracer.py:58-70) on the
host cores (pthreads).  Returns plain numpy record/path dicts.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "libtracer_oracle.so")
S, E, M = 32, 16, 8
d, i32, i64 = C.c_double, C.c_int32, C.c_int64


def _a(t, *dims):
    for n in reversed(dims):
        t = t * n
    return t


class OScene(C.Structure):
    _fields_ = [("ns", C.c_int), ("ne", C.c_int), ("nm", C.c_int), ("width", C.c_int),
                ("height", C.c_int), ("stype", _a(C.c_int, S)), ("mat", _a(C.c_int, S)),
                ("emid", _a(C.c_int, S)), ("sp", _a(d, S, 9)), ("alb", _a(d, S, 3)),
                ("etype", _a(C.c_int, E)), ("eval", _a(d, E, 3)), ("epos", _a(d, E, 3)),
                ("equad", _a(d, E, 9)), ("enrm", _a(d, E, 3)), ("earea", _a(d, E)),
                ("mkind", _a(C.c_int, M)), ("dims", _a(C.c_int, M, 3)), ("st", _a(d, M, 3)),
                ("ss", _a(d, M, 3)), ("mg", _a(d, M)), ("mb", _a(d, M, 6)), ("mu", _a(d, M)),
                ("mscale", _a(d, M)), ("goff", _a(i64, M)), ("grid", C.c_void_p),
                ("cam", _a(d, 15))]


REC = [("pos", 3, np.float64), ("omega_out", 3, np.float64), ("normal", 3, np.float64),
       ("coeff", 3, np.float64), ("g", 1, np.float64), ("phase_dir", 3, np.float64),
       ("pdf_phase", 1, np.float64), ("pdf_emit_at_phase", 1, np.float64),
       ("emit_dir", 3, np.float64), ("pdf_emit", 1, np.float64), ("d_emit", 3, np.float64),
       ("d_phase", 3, np.float64), ("i_pt", 3, np.float64), ("w_cont", 3, np.float64),
       ("kind", 1, np.uint8), ("emit_delta", 1, np.uint8), ("class_id", 1, np.int32),
       ("path_idx", 1, np.int64), ("depth", 1, np.int32)]
PTH = ["cam_weight", "d_cam", "direct0", "direct0_nee", "direct0_phase", "pt_estimate"]


class ORec(C.Structure):
    _fields_ = [(n, C.c_void_p) for n, _, _ in REC]


class OPath(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in PTH]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-s", "-C", HERE], check=True)
        _lib = C.CDLL(LIB)
        assert _lib.oracle_scene_size() == C.sizeof(OScene)
    return _lib


def flatten(scene):
    """Reference flattening (flatten.py:87-195) into the oracle's struct."""
    st = OScene()
    st.ns, st.ne, st.nm = len(scene.surfaces), len(scene.emitters), len(scene.media)
    codes = {"sphere": 0, "box": 1, "quad": 2}
    mats = {"lambertian": 0, "black": 1, "emitter": 2}
    for k, s in enumerate(scene.surfaces):
        st.stype[k], st.mat[k], st.emid[k] = codes[s.geometry], mats[s.material], s.emitter_index
        for a, p in enumerate(s.params):
            st.sp[k][a] = p
        for a in range(3):
            st.alb[k][a] = s.albedo[a]
    for j, e in enumerate(scene.emitters):
        for a in range(3):
            st.eval[j][a] = e.value[a]
        if e.kind == "point":
            st.etype[j] = 0
            for a in range(3):
                st.epos[j][a] = e.position[a]
        elif e.kind == "directional":
            st.etype[j] = 2
            v = np.asarray(e.direction, dtype=np.float64)
            v = v / np.linalg.norm(v)
            for a in range(3):
                st.epos[j][a] = v[a]
        else:
            st.etype[j] = 1
            q = next(s.params for s in scene.surfaces
                     if s.material == "emitter" and s.emitter_index == j)
            for a in range(9):
                st.equad[j][a] = q[a]
            u, v = np.asarray(q[3:6], np.float64), np.asarray(q[6:9], np.float64)
            st.earea[j] = float(np.linalg.norm(np.cross(u, v)))
            x = u[1] * v[2] - u[2] * v[1]
            y = u[2] * v[0] - u[0] * v[2]
            z = u[0] * v[1] - u[1] * v[0]
            inv = 1.0 / math.sqrt(x * x + y * y + z * z)
            st.enrm[j][0], st.enrm[j][1], st.enrm[j][2] = x * inv, y * inv, z * inv
    chunks, off = [], 0
    for k, m in enumerate(scene.media):
        st.mkind[k] = 0 if m.kind == "homogeneous" else 1
        for a in range(3):
            st.st[k][a], st.ss[k][a] = m.sigma_t[a], m.sigma_s[a]
        st.mg[k] = m.phase_g
        for a in range(6):
            st.mb[k][a] = m.bounds[a]
        st.mscale[k] = m.density_scale
        if m.kind == "grid":
            vol = np.ascontiguousarray(m.density, dtype=np.float32)
            nz, ny, nx = vol.shape
            st.dims[k][0], st.dims[k][1], st.dims[k][2] = nx, ny, nz
            st.goff[k] = off
            chunks.append(vol.ravel())
            off += vol.size
            st.mu[k] = float(vol.max()) * m.density_scale * float(max(m.sigma_t))
        else:
            st.mu[k] = float(max(m.sigma_t))
    grid = np.concatenate(chunks) if chunks else np.zeros(1, np.float32)
    st.grid = grid.ctypes.data
    cam = scene.camera
    org = np.asarray(cam.origin, np.float64)
    fwd = np.asarray(cam.look_at, np.float64) - org
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(cam.up, np.float64))
    nrm = np.linalg.norm(right)
    if nrm < 1e-9:
        right = np.cross(fwd, np.array([1.0, 0.0, 0.0]))
        nrm = np.linalg.norm(right)
    right /= nrm
    up = np.cross(right, fwd)
    w, h = cam.resolution
    vals = list(org) + list(fwd) + list(right) + list(up) + \
        [float(np.tan(np.radians(cam.fov) * 0.5)), float(w), float(h)]
    for a, v in enumerate(vals):
        st.cam[a] = v
    st.width, st.height = w, h
    return st, grid


def trace_records(scene, cfg):
    """(records dict, paths dict) of an instrumented render, CPU only."""
    L = lib()
    st, grid = flatten(scene)
    spp = int(cfg.spp)
    n_paths = st.width * st.height * spp
    args = (C.byref(st), C.c_int(spp), C.c_int(int(cfg.max_depth)), C.c_int(int(cfg.rr_start)),
            C.c_double(float(cfg.rr_floor)), C.c_int64(int(np.int64(cfg.seed))))
    counts = np.zeros(n_paths, dtype=np.int64)
    threads = C.c_int(os.cpu_count() or 1)
    L.oracle_trace_count(*args, C.c_void_p(counts.ctypes.data), threads)
    offsets = np.zeros(n_paths, dtype=np.int64)
    np.cumsum(counts[:-1], out=offsets[1:])
    n = int(counts.sum())
    rec = {name: np.zeros((n, w) if w > 1 else n, dtype=dt) for name, w, dt in REC}
    r = ORec(*[rec[name].ctypes.data for name, _, _ in REC])
    paths = {name: np.zeros((n_paths, 3)) for name in PTH}
    p = OPath(*[paths[name].ctypes.data for name in PTH])
    L.oracle_trace_fill(*args, C.c_void_p(offsets.ctypes.data), C.byref(r), C.byref(p), threads)
    paths["pixel_idx"] = np.arange(n_paths, dtype=np.int64) // spp
    paths["rec_start"] = offsets
    paths["rec_count"] = counts.astype(np.int32)
    paths["extra_direct"] = paths["direct0"].copy()
    del grid
    return rec, paths

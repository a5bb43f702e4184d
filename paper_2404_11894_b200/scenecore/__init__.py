"""Scene description (host-side setup for the CUDA tracer).

Names mirror the reference's scenecore package (scenecore/__init__.py:1-35)
for everything a caller constructs; the per-sample njit helpers of the
reference (eval_phase, sample_distance, ...) are device functions here.
"""

from paper_2404_11894_b200.scenecore.types import (
    Camera,
    Emitter,
    Medium,
    PhaseHG,
    Scene,
    SceneError,
    Surface,
    as_spectrum,
    make_camera,
)
from paper_2404_11894_b200.scenecore.volgrid import read_volume_grid, write_volume_grid

__all__ = [
    "Camera",
    "Emitter",
    "Medium",
    "PhaseHG",
    "Scene",
    "SceneError",
    "Surface",
    "as_spectrum",
    "make_camera",
    "read_volume_grid",
    "write_volume_grid",
]

"""B200-native path-graph renderer (arXiv 2404.11894), a drop-in for the
reference `volpg` package's render / path-graph API.

    import paper_2404_11894_b200 as volpg
    from paper_2404_11894_b200.pathgraph import build_graph, solve, splat_output

Compute runs in libvolpg_b200.so (hand-written sm_100a CUDA, C ABI in
include/volpg_b200.h); there is no CPU fallback.
"""

__version__ = "0.1.0"

from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.scenecore.types import (Camera, Emitter, Medium, PhaseHG, Scene,
                                                   SceneError, Surface)

__all__ = [
    "Camera",
    "Emitter",
    "Medium",
    "PhaseHG",
    "RenderConfig",
    "Scene",
    "SceneError",
    "Surface",
]

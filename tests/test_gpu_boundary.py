"""The drop-in boundary with the reference's own objects and bindings.

- reconstruct_path_estimate (transport/reconstruct.py:52-72) on the device:
  the records of a path rebuild its PT estimate to 1e-5, on
  the reference's record sets (goldens) and on device-traced ones.
- duck-typed reference objects: a volpg-style TraceOutput / RecordSoA /
  PathSoA (plain attribute bags here: the reference is not installed on the
  GPU box) through build_graph / solve_from_records, a volpg-style Scene and
  RenderConfig through render_pg.
- the ctypes shim of INTEGRATION.md §2, executed verbatim.
"""

import os
import re
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import ROOT, assert_rel, golden
from oracle import pathgraph_oracle as O

pytestmark = pytest.mark.gpu

REC = ["pos", "omega_out", "normal", "coeff", "g", "phase_dir", "pdf_phase", "pdf_emit_at_phase",
       "emit_dir", "pdf_emit", "d_emit", "d_phase", "i_pt", "w_cont", "kind", "emit_delta",
       "class_id", "path_idx", "depth"]
PTH = ["pixel_idx", "rec_start", "rec_count", "cam_weight", "d_cam", "direct0", "direct0_nee",
       "direct0_phase", "extra_direct", "pt_estimate"]


def _ref_like_trace(z):
    """An object shaped like volpg's TraceOutput (records.py:179-188), not ours."""
    rec, paths = O.load_golden_records(z)
    r = SimpleNamespace(**{f: rec[f] for f in REC}, n=rec["pos"].shape[0],
                        cluster_id=np.full(rec["pos"].shape[0], -1, np.int64))
    p = SimpleNamespace(**{f: paths[f] for f in PTH}, n=paths["rec_start"].shape[0])
    return SimpleNamespace(image=z["pt_image"], records=r, paths=p, width=int(z["width"]),
                           height=int(z["height"]), spp=int(z["spp"]))


def _pt_scale(est):
    return np.maximum(np.abs(est), 1e-5 * float(np.abs(est).max()) + 1e-300)


@pytest.mark.parametrize("name", ["c1_16", "c1floor_16", "cloud_16", "mixed_12", "dense_12"])
def test_reconstruct_reference_records(cuda, name):
    from paper_2404_11894_b200.transport import reconstruct_path_estimates

    z = golden(name)
    t = _ref_like_trace(z)
    est, diff = reconstruct_path_estimates(t.records, t.paths)
    ref = t.paths.pt_estimate
    err = np.abs(est - ref) / _pt_scale(ref)
    assert float(err.max()) <= 1e-5, (name, float(err.max()))
    ipt_scale = float(np.abs(t.records.i_pt).max()) + 1e-300
    assert float(diff.max()) <= 1e-5 * ipt_scale


@pytest.mark.parametrize("factory", ["c1", "mixed", "c2"])
def test_reconstruct_device_traced_records(cuda, factory):
    """SPEC.md:197 on the device tracer's own records and estimates."""
    from paper_2404_11894_b200 import scenes as S
    from paper_2404_11894_b200.harness.config import RenderConfig
    from paper_2404_11894_b200.transport import (reconstruct_path_estimate,
                                                 reconstruct_path_estimates, render_pt)

    scene = {"c1": lambda: S.scene_c1((32, 32), floor=True), "mixed": lambda: S.scene_mixed((24, 24)),
             "c2": lambda: S.scene_c2((32, 32), grid_n=64)}[factory]()
    out = render_pt(scene, RenderConfig(spp=4, max_depth=64, seed=3), with_records=True)
    est, diff = reconstruct_path_estimates(out.records, out.paths)
    ref = out.paths.pt_estimate
    err = np.abs(est - ref) / _pt_scale(ref)
    assert float(err.max()) <= 1e-5, float(err.max())
    assert float(diff.max()) <= 1e-5 * (float(np.abs(out.records.i_pt).max()) + 1e-300)
    i = int(np.argmax(out.paths.rec_count))
    one, d1 = reconstruct_path_estimate(out.records, out.paths, i)
    assert np.array_equal(one, est[i]) and d1 == diff[i]
    with pytest.raises(IndexError):
        reconstruct_path_estimate(out.records, out.paths, out.paths.n)


def test_reference_trace_objects(cuda):
    """build_graph / solve / splat_output and solve_from_records on a
    volpg-shaped TraceOutput: same results as the reference, and
    records.cluster_id written back into it (graph.py:62)."""
    from paper_2404_11894_b200.pathgraph import build_graph, solve, splat_output
    from paper_2404_11894_b200.pathgraph.pipeline import solve_from_records

    z = golden("c1floor_16")
    t = _ref_like_trace(z)
    g = build_graph(t, 32, seed=int(z["seed"]))
    assert np.array_equal(t.records.cluster_id, z["K32_cluster_id"])
    res = solve(g, iterations=10, tol=0.0)
    assert_rel(res.incoming, z["K32_it10_incoming"], 1e-4, what="incoming")
    assert_rel(splat_output(g, res), z["K32_it10_image"], 1e-4, what="image")
    t2 = _ref_like_trace(z)
    img, g2, r2 = solve_from_records(t2, 32, iterations=10, tol=0.0, seed=int(z["seed"]))
    assert np.array_equal(t2.records.cluster_id, z["K32_cluster_id"])
    assert_rel(img, z["K32_it10_image"], 1e-4, what="solve_from_records image")


def _plain(obj):
    """A volpg-shaped copy of one of our scene objects: same field names,
    different classes (attribute bags)."""
    from dataclasses import fields, is_dataclass

    if is_dataclass(obj):
        return SimpleNamespace(**{f.name: _plain(getattr(obj, f.name)) for f in fields(obj)})
    if isinstance(obj, list):
        return [_plain(x) for x in obj]
    return obj


def test_reference_scene_and_config_objects(cuda):
    from paper_2404_11894_b200 import scenes as S
    from paper_2404_11894_b200.harness.config import RenderConfig
    from paper_2404_11894_b200.pathgraph import render_pg

    scene = S.scene_mixed((16, 16))
    cfg = RenderConfig(mode="pg", spp=2, max_depth=32, seed=4, iterations=6, tol=0.0)
    ours = render_pg(scene, cfg)
    theirs = render_pg(_plain(scene), SimpleNamespace(**vars(cfg)))
    assert np.array_equal(ours.image, theirs.image)
    assert np.array_equal(ours.pt_image, theirs.pt_image)


def test_integration_shim_verbatim(cuda):
    """INTEGRATION.md §2, executed as written: the reference's RecordSoA and
    the Generator graph.py:60 creates go in; the clusters, the Generator's
    state afterwards and the solve match the reference."""
    import torch

    from paper_2404_11894_b200 import _native as N

    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = re.search(r"## 2\..*?```python\n(.*?)```", text, re.S).group(1)
    os.environ["VOLPG_B200_LIB"] = N.LIB_PATH
    ns = {}
    exec(compile(block, "INTEGRATION.md#2", "exec"), ns)
    z = golden("cloud_16")
    t = _ref_like_trace(z)
    seed = int(z["seed"])
    rng = np.random.default_rng(np.random.SeedSequence([seed & 0xFFFFFFFF, 0xC1A5]))
    g, dev = ns["build_graph_b200"](t.records, 32, rng)
    ref_rng = np.random.default_rng(np.random.SeedSequence([seed & 0xFFFFFFFF, 0xC1A5]))
    O.cluster_points(t.records.pos, O.class_keys(t.records.kind, t.records.class_id), 32, ref_rng)
    assert rng.bit_generator.state == ref_rng.bit_generator.state
    incoming, i_bar, res = ns["solve_b200"](g, t.records.n, 10, 0.0)
    torch.cuda.synchronize()
    assert_rel(incoming, z["K32_it10_incoming"], 1e-4, what="incoming")
    assert_rel(i_bar, z["K32_it10_i_bar"], 1e-4, what="i_bar")
    np.testing.assert_allclose(res, z["K32_it10_residuals"], rtol=1e-4, atol=1e-6)
    ns["_lib"].vpg_graph_free(g)

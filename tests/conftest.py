import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the native kernels")


def golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def assert_rel(got, ref, rtol, floor=1e-30, what=""):
    """Per entry |got-ref| <= rtol*|ref| (+ a denormal floor), zeros exact."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    err = np.abs(got - ref)
    bad = err > rtol * np.abs(ref) + floor
    assert not bad.any(), (
        f"{what}: {int(bad.sum())} entries outside rtol={rtol}; worst rel "
        f"{float((err / np.maximum(np.abs(ref), 1e-300)).max()):.3e}")
    zero = ref == 0.0
    assert np.all(got[zero] == 0.0), f"{what}: {int((got[zero] != 0).sum())} nonzeros where ref == 0"


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return torch


# ---------------------------------------------------------------- scale goldens
SCALE_CASES = ["c1_s0", "c1_s1", "c1_s2", "c2_slice", "c3_slice", "c4_slice"]
_SCALE_SCENES = {  # must match tests/golden/make_golden_scale.py
    "c1_s0": ("scene_c1", (64, 64)), "c1_s1": ("scene_c1", (64, 64)),
    "c1_s2": ("scene_c1", (64, 64)), "c2_slice": ("scene_c2", (96, 96)),
    "c3_slice": ("scene_c3", (64, 64)), "c4_slice": ("scene_c4", (96, 96)),
}
_scale_cache = {}


def sha64(a) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def scale_case(name):
    """(fixture, records, paths): the reference's own record set of a scale
    case, rebuilt by the oracle's C tracer plus the committed XOR patch and
    checked field by field against the reference's sha256."""
    if name in _scale_cache:
        return _scale_cache[name]
    import hashlib

    from oracle import tracer_oracle as T
    from paper_2404_11894_b200 import scenes as S
    from paper_2404_11894_b200.harness.config import RenderConfig

    z = dict(np.load(os.path.join(GOLDEN, f"scale_{name}.npz")))
    fac, res = _SCALE_SCENES[name]
    cfg = RenderConfig(spp=int(z["spp"]), max_depth=int(z["max_depth"]), seed=int(z["seed"]))
    rec, paths = T.trace_records(getattr(S, fac)(res), cfg)
    for f in list(rec):
        x = z["xrec_" + f]
        a = np.ascontiguousarray(rec[f])
        rec[f] = (a.view(x.dtype) ^ x).view(a.dtype).reshape(a.shape)
        assert hashlib.sha256(rec[f].tobytes()).hexdigest() == str(z["sha_rec_" + f]), f
    for k in list(z):
        if k.startswith("xpath_"):
            f = k[6:]
            a = np.ascontiguousarray(paths[f])
            paths[f] = (a.view(z[k].dtype) ^ z[k]).view(a.dtype).reshape(a.shape)
    paths["extra_direct"] = paths["direct0"].copy()
    _scale_cache.clear()  # one big case at a time
    _scale_cache[name] = (z, rec, paths)
    return _scale_cache[name]


def csr_topology_hashes(cluster_id, off, members):
    """sha256 of the reference CSR's indptr / indices (graph.py:167: row r holds
    its cluster's members, ascending), computed from the clusters in row
    chunks."""
    import hashlib

    sizes = np.diff(off)
    row_size = sizes[cluster_id]
    indptr = np.zeros(cluster_id.shape[0] + 1, np.int64)
    np.cumsum(row_size, out=indptr[1:])
    h = hashlib.sha256()
    step = 1 << 18
    for b in range(0, cluster_id.shape[0], step):
        c = cluster_id[b:b + step]
        st, ln = off[c], sizes[c]
        tot = int(ln.sum())
        base = np.repeat(st - (np.cumsum(ln) - ln), ln)
        h.update(members[base + np.arange(tot)].astype(np.int64).tobytes())
    return sha64(indptr), h.hexdigest()

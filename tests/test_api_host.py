"""Host-side API behaviour of the reference surface (no GPU): argument checks
and their exception types, the residual norm, the residual CSV, scene
validation, and the error mapping of the C ABI."""

import csv

import numpy as np
import pytest

from oracle import pathgraph_oracle as O
from paper_2404_11894_b200 import _native as N
from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.pathgraph import residual_norm, write_residual_csv
from paper_2404_11894_b200.pathgraph.solve import SolveDivergence


def test_residual_norm_matches_reference_definition():
    rs = np.random.default_rng(0)
    new, old = rs.random((50, 3)), rs.random((50, 3))
    want = max(np.abs(new[:, c] - old[:, c]).max() / max(np.abs(new[:, c]).max(), 1e-12)
               for c in range(3))
    assert residual_norm(new, old) == want
    assert residual_norm(np.zeros((4, 3)), np.zeros((4, 3))) == 0.0
    assert residual_norm(np.zeros((0, 3)), np.zeros((0, 3))) == 0.0


def test_residual_norm_agrees_with_oracle_on_nan():
    new = np.array([[np.nan, 1.0, 2.0], [0.5, 0.5, 0.5]])
    old = np.zeros((2, 3))
    assert residual_norm(new, old) == O.residual_norm(new, old)


def test_write_residual_csv_format(tmp_path):
    path = tmp_path / "res.csv"
    write_residual_csv(str(path), [0.5, 0.125, 1e-17])
    rows = list(csv.reader(open(path)))
    assert rows == [["iteration", "residual"], ["1", "0.5"], ["2", "0.125"], ["3", "1e-17"]]


@pytest.mark.parametrize("kw", [dict(spp=0), dict(cluster_size=0), dict(iterations=-1),
                                dict(max_depth=0), dict(rr_floor=0.0), dict(mode="nope")])
def test_render_config_rejects_bad_values(kw):
    with pytest.raises(ValueError):
        RenderConfig(**kw)


def test_solve_divergence_is_a_runtime_error():
    assert issubclass(SolveDivergence, RuntimeError)


def test_native_error_codes_map_to_reference_exceptions():
    lib = N.lib()
    st = N.Pcg64State.from_generator(np.random.default_rng(0))
    out = np.zeros(4, np.int64)
    # choice with m > n is a ValueError in numpy (and here)
    with pytest.raises(ValueError):
        N.check(lib.vpg_rng_choice(st, 3, 4, out.ctypes.data))
    with pytest.raises(SolveDivergence):
        N.check(N.VPG_EDIVERGED)
    with pytest.raises(MemoryError):
        N.check(N.VPG_ENOMEM)

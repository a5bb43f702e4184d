"""The harness around the device pipeline (the reference
declares the CLI and runners but ships only pfm / metrics): PFM round trips,
MSE, the CLI's error handling on CPU; render / iteration study on the GPU."""

import os

import numpy as np
import pytest

from paper_2404_11894_b200.harness import PfmError, compute_mse, read_pfm, write_pfm
from paper_2404_11894_b200.harness.cli import main


def test_pfm_round_trip_is_bit_exact(tmp_path):
    rs = np.random.default_rng(0)
    img = rs.random((7, 5, 3)).astype(np.float32) * 10
    img[0, 0] = [0.0, np.float32(1e-38), np.float32(3.4e38)]
    p = tmp_path / "a.pfm"
    write_pfm(img, p)
    back = read_pfm(p)
    assert back.dtype == np.float32 and back.shape == img.shape
    assert back.tobytes() == img.tobytes()
    raw = open(p, "rb").read()
    assert raw.startswith(b"PF\n5 7\n-1.0\n")
    # rows are stored bottom to top
    assert raw[-12:] == img[0, -1].astype("<f4").tobytes()


def test_pfm_errors(tmp_path):
    p = tmp_path / "bad.pfm"
    p.write_bytes(b"P6\n1 1\n255\n\0\0\0")
    with pytest.raises(PfmError):
        read_pfm(p)
    p.write_bytes(b"PF\n2 2\n-1.0\n" + b"\0" * 20)
    with pytest.raises(PfmError):
        read_pfm(p)
    p.write_bytes(b"PF\n1 1\n1.0\n" + b"\0" * 12)
    with pytest.raises(PfmError):
        read_pfm(p)
    with pytest.raises(PfmError):
        write_pfm(np.zeros((2, 2)), tmp_path / "x.pfm")


def test_mse_matches_scalar_loop():
    rs = np.random.default_rng(1)
    a, b = rs.random((6, 4, 3)), rs.random((6, 4, 3))
    s = 0.0
    for v, w in zip(a.ravel(), b.ravel()):
        s += (v - w) ** 2
    assert abs(compute_mse(a, b) - s / a.size) <= 1e-12
    assert compute_mse(a, a) == 0.0
    assert abs(compute_mse(np.zeros((2, 2, 3)), np.full((2, 2, 3), 0.1)) - 0.01) < 1e-15
    with pytest.raises(ValueError):
        compute_mse(a, b[:5])


def test_cli_mse_and_errors(tmp_path, capsys):
    a, b = tmp_path / "a.pfm", tmp_path / "b.pfm"
    write_pfm(np.zeros((2, 3, 3)), a)
    write_pfm(np.full((2, 3, 3), 0.5), b)
    assert main(["mse", str(a), str(b)]) == 0
    assert float(capsys.readouterr().out) == 0.25
    assert main(["mse", str(a), str(tmp_path / "missing.pfm")]) != 0
    assert main(["render", "--scene", "nope"]) != 0


@pytest.mark.gpu
def test_cli_render_and_iteration_study(cuda, tmp_path, capsys):
    from paper_2404_11894_b200 import scenes as S
    from paper_2404_11894_b200.harness.config import RenderConfig
    from paper_2404_11894_b200.harness.experiments import run_iteration_study
    from paper_2404_11894_b200.pathgraph import render_pg

    out = tmp_path / "pg.pfm"
    assert main(["render", "--scene", "C1", "--res", "16x16", "--mode", "pg", "--spp", "2",
                 "--seed", "3", "--out", str(out)]) == 0
    cfg = RenderConfig(mode="pg", spp=2, seed=3)
    ref = render_pg(S.WORKLOADS["C1"].scene((16, 16)), cfg).image
    assert read_pfm(out).tobytes() == ref.astype(np.float32).tobytes()
    # determinism: the same command line gives the same bytes
    out2 = tmp_path / "pg2.pfm"
    main(["render", "--scene", "C1", "--res", "16x16", "--mode", "pg", "--spp", "2",
          "--seed", "3", "--out", str(out2)])
    assert open(out, "rb").read() == open(out2, "rb").read()
    # iteration study: 0 iterations is the initialisation, rows pair with images
    images, rows = run_iteration_study(S.WORKLOADS["C1"].scene((16, 16)), cfg, [0, 1, 10],
                                       csv_path=str(tmp_path / "it.csv"))
    assert [r[0] for r in rows] == [0, 1, 10] and len(images) == 3
    assert len(open(tmp_path / "it.csv").read().strip().splitlines()) == 4

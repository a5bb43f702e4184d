"""Experiment runners over the device pipeline (declared by the reference,
SPEC.md:390-409, but missing there): error-vs-spp convergence of PT and the
path graph against a high-spp PT reference, and the iteration study on one
traced record set."""

from __future__ import annotations

import csv
import dataclasses
import time

import numpy as np

from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.harness.metrics import compute_mse


def render_reference(scene, config: RenderConfig, spp: int) -> np.ndarray:
    """mode=reference: PT at high spp, records off."""
    from paper_2404_11894_b200.transport import render_pt

    cfg = dataclasses.replace(config, mode="reference", spp=int(spp))
    return render_pt(scene, cfg).image


def run_convergence(scene, config: RenderConfig, spp_list, seeds, reference,
                    csv_path=None) -> list:
    """Rows (method, spp, seed, mse, wall_seconds) for pt and pg at every spp
    and seed, against `reference` (an image)."""
    from paper_2404_11894_b200.pathgraph import render_pg
    from paper_2404_11894_b200.transport import render_pt

    rows = []
    for spp in spp_list:
        for seed in seeds:
            cfg = dataclasses.replace(config, spp=int(spp), seed=int(seed))
            t0 = time.perf_counter()
            pt = render_pt(scene, dataclasses.replace(cfg, mode="pt")).image
            t1 = time.perf_counter()
            pg = render_pg(scene, dataclasses.replace(cfg, mode="pg")).image
            t2 = time.perf_counter()
            rows.append(("pt", int(spp), int(seed), compute_mse(pt, reference), t1 - t0))
            rows.append(("pg", int(spp), int(seed), compute_mse(pg, reference), t2 - t1))
    if csv_path:
        with open(csv_path, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["method", "spp", "seed", "mse", "wall_seconds"])
            for r in rows:
                w.writerow([r[0], r[1], r[2], repr(r[3]), repr(r[4])])
    return rows


def run_iteration_study(scene, config: RenderConfig, iteration_list, reference=None,
                        csv_path=None) -> tuple:
    """One traced record set, one graph, a solve per iteration count: the
    images and (iterations, mse, residual) rows (mse None without a
    reference).  0 iterations gives the PT image (the initialisation)."""
    from paper_2404_11894_b200.pathgraph import build_graph, solve, splat_output
    from paper_2404_11894_b200.transport import render_pt

    trace = render_pt(scene, config, with_records=True)
    graph = build_graph(trace, config.cluster_size, seed=config.seed)
    images, rows = [], []
    for it in iteration_list:
        res = solve(graph, iterations=int(it), tol=0.0)
        img = splat_output(graph, res, aggregate_direct_term=config.aggregate_direct)
        images.append(img)
        mse = compute_mse(img, reference) if reference is not None else None
        resid = res.residuals[-1] if res.residuals else None
        rows.append((int(it), mse, resid))
    if csv_path:
        with open(csv_path, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["iterations", "mse", "residual"])
            for r in rows:
                w.writerow([r[0], "" if r[1] is None else repr(r[1]),
                            "" if r[2] is None else repr(r[2])])
    return images, rows

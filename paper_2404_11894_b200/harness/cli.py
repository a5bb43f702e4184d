"""Command line over the device pipeline (the reference declares
`volpg render|mse|convergence|iterations`, pyproject.toml:20,
but ships no cli module).  Scenes are the built-in configurations (C1-C5 of
BASELINE.json, `mixed`, and the SPEC.md acceptance scenes `fogbox` and
`gridpuff`); images are written as PFM.

    python -m paper_2404_11894_b200.harness.cli render --scene C1 --mode pg --spp 4 --out pg.pfm
    python -m paper_2404_11894_b200.harness.cli mse pg.pfm ref.pfm
    python -m paper_2404_11894_b200.harness.cli convergence --scene C1 --spp-list 1,4 --seeds 0 \\
        --reference-spp 256 --csv conv.csv
    python -m paper_2404_11894_b200.harness.cli iterations --scene C1 --iteration-list 0,1,10 \\
        --csv it.csv
"""

from __future__ import annotations

import argparse
import sys

from paper_2404_11894_b200.harness.config import RenderConfig


def _scene(name: str, res):
    from paper_2404_11894_b200 import scenes as S

    if name == "mixed":
        return S.scene_mixed(res or (12, 12))
    if name == "fogbox":
        return S.scene_fogbox(res or (128, 128))
    if name == "gridpuff":
        return S.scene_gridpuff(res or (256, 256))
    if name not in S.WORKLOADS:
        raise ValueError(f"unknown scene {name!r} (C1-C5, mixed, fogbox or gridpuff)")
    return S.WORKLOADS[name].scene(res)


def _res(text):
    if not text:
        return None
    w, h = (int(v) for v in text.lower().split("x"))
    return (w, h)


def _ints(text):
    return [int(v) for v in text.split(",") if v.strip()]


def _config(a) -> RenderConfig:
    return RenderConfig(mode=a.mode, spp=a.spp, seed=a.seed, cluster_size=a.cluster_size,
                        iterations=a.iterations, tol=a.tol, max_depth=a.max_depth,
                        extra_direct_samples=a.extra_direct, aggregate_direct=a.aggregate_direct,
                        dump_records=a.dump_records, residual_csv=a.residual_csv, out=a.out)


def _add_render_args(p):
    p.add_argument("--scene", default="C1")
    p.add_argument("--res", default=None, help="override the resolution, WxH")
    p.add_argument("--mode", default="pg", choices=["pt", "pg", "reference"])
    p.add_argument("--spp", type=int, default=1)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--cluster-size", type=int, default=32)
    p.add_argument("--iterations", type=int, default=10)
    p.add_argument("--tol", type=float, default=1e-3)
    p.add_argument("--max-depth", type=int, default=64)
    p.add_argument("--extra-direct", type=int, default=0)
    p.add_argument("--aggregate-direct", action="store_true")
    p.add_argument("--dump-records", default=None)
    p.add_argument("--residual-csv", default=None)
    p.add_argument("--out", default=None)


def cmd_render(a) -> int:
    from paper_2404_11894_b200.harness.pfm import write_pfm
    from paper_2404_11894_b200.pathgraph import render_pg
    from paper_2404_11894_b200.transport import render_pt, save_records

    cfg = _config(a)
    scene = _scene(a.scene, _res(a.res))
    if cfg.mode == "pg":
        image = render_pg(scene, cfg).image
    else:
        out = render_pt(scene, cfg, with_records=bool(cfg.dump_records))
        if cfg.dump_records:
            save_records(cfg.dump_records, out)
        image = out.image
    if cfg.out:
        write_pfm(image, cfg.out)
    print(f"{cfg.mode}: {image.shape[1]}x{image.shape[0]}, mean {float(image.mean()):.6g}")
    return 0


def cmd_mse(a) -> int:
    from paper_2404_11894_b200.harness.metrics import compute_mse
    from paper_2404_11894_b200.harness.pfm import read_pfm

    print(repr(compute_mse(read_pfm(a.image), read_pfm(a.reference))))
    return 0


def cmd_convergence(a) -> int:
    from paper_2404_11894_b200.harness.experiments import render_reference, run_convergence

    cfg = _config(a)
    scene = _scene(a.scene, _res(a.res))
    ref = render_reference(scene, cfg, a.reference_spp)
    for r in run_convergence(scene, cfg, _ints(a.spp_list), _ints(a.seeds), ref, a.csv):
        print(",".join(str(v) for v in r))
    return 0


def cmd_iterations(a) -> int:
    from paper_2404_11894_b200.harness.experiments import render_reference, run_iteration_study
    from paper_2404_11894_b200.harness.pfm import write_pfm

    cfg = _config(a)
    scene = _scene(a.scene, _res(a.res))
    ref = render_reference(scene, cfg, a.reference_spp) if a.reference_spp else None
    iters = _ints(a.iteration_list)
    images, rows = run_iteration_study(scene, cfg, iters, ref, a.csv)
    if a.out_prefix:
        for it, img in zip(iters, images):
            write_pfm(img, f"{a.out_prefix}_it{it}.pfm")
    for r in rows:
        print(",".join("" if v is None else str(v) for v in r))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="volpg-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("render")
    _add_render_args(p)
    p = sub.add_parser("mse")
    p.add_argument("image")
    p.add_argument("reference")
    p = sub.add_parser("convergence")
    _add_render_args(p)
    p.add_argument("--spp-list", default="1,4,16")
    p.add_argument("--seeds", default="0")
    p.add_argument("--reference-spp", type=int, default=1024)
    p.add_argument("--csv", default=None)
    p = sub.add_parser("iterations")
    _add_render_args(p)
    p.add_argument("--iteration-list", default="0,1,2,5,10,20")
    p.add_argument("--reference-spp", type=int, default=0)
    p.add_argument("--csv", default=None)
    p.add_argument("--out-prefix", default=None)
    a = ap.parse_args(argv)
    handler = {"render": cmd_render, "mse": cmd_mse, "convergence": cmd_convergence,
               "iterations": cmd_iterations}[a.cmd]
    try:
        return handler(a)
    except (ValueError, IOError, RuntimeError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())

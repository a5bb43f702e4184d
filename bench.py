#!/usr/bin/env python
"""Benchmark: graph vertices propagated/s (build + K iterations) and ms/frame.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]
                    [--workload C2] [--cpu-sample 96]

One step = one pass of the hot path over the workload's record set already
resident in HBM: build_graph (exact clustering, marginals, operator blocks)
+ solve(iterations=K_iter, tol=0).  `value` = vertices * N / step time.
`e2e` = the same metric through the reference-facing API with HOST buffers
(solve_from_records on pinned host records: H2D, build, solve, splat, image
D2H inside the timed region).  The workload (BASELINE.json configs[1] = C2)
is traced by the CUDA tracer once, outside the timed region; the synthetic
fbm cloud is procedural (no dataset).  Inputs (2.4 GB of records, 1.2 GB of
kernel blocks) are far larger than the 126 MB L2.

--impl reference times the reference algorithm's CPU restatement (oracle/,
numpy) on a bounded sample of the same workload traced by the oracle's C
tracer restatement, on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "graph vertices propagated/sec (build+K iters) and ms/frame at 1/2/4/8 B200"
UNIT = "vertices/s"
# SURVEY.md §8d algorithmic bytes per vertex (fp32 values, int32 indices,
# fp64 positions, CSR W with nnz/N = 36.5)
BUILD_BYTES_PER_VERTEX = 632
ITER_BYTES_PER_VERTEX = 360


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--cpu-sample", type=int, default=64,
                    help="square resolution of the CPU-baseline sample of the workload")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during timing."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={','.join(self.FIELDS)}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------- helpers
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_config(name):
    from paper_2404_11894_b200.harness.config import RenderConfig
    from paper_2404_11894_b200.scenes import WORKLOADS

    wl = WORKLOADS[name]
    cfg = RenderConfig(mode="pg", spp=wl.spp, seed=0, cluster_size=32, iterations=wl.iterations,
                       tol=0.0, max_depth=wl.max_depth)
    return wl, cfg


def cpu_baseline(wl, cfg, sample_res, trace_fn, steps=1):
    """The oracle (numpy restatement of the reference) on a bounded sample."""
    from oracle import pathgraph_oracle as O

    scene = wl.scene((sample_res, sample_res))
    rec, paths = trace_fn(scene, cfg)
    n = rec["pos"].shape[0]
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        g = O.build_graph(rec, paths, sample_res, sample_res, cfg.spp, cfg.cluster_size, cfg.seed)
        O.solve(g, cfg.iterations, 0.0)
        times.append(time.perf_counter() - t0)
    t = min(times)
    return {"value": n / t, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{wl.name} scene at {sample_res}x{sample_res}, {cfg.spp} spp: {n} vertices, "
                      f"build + {cfg.iterations} iterations in {t:.2f} s (oracle/pathgraph_oracle.py, "
                      f"numpy, best of {steps})"}, n, t


def device_trace_sample(scene, cfg):
    from paper_2404_11894_b200.transport import render_pt

    out = render_pt(scene, cfg, with_records=True)
    return out.records.host_arrays(), out.paths.host_arrays()


def oracle_trace_sample(scene, cfg):
    from oracle import tracer_oracle

    return tracer_oracle.trace_records(scene, cfg)


# ------------------------------------------------------------ reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    wl, cfg = workload_config(args.workload)
    res = args.cpu_sample
    scene = wl.scene((res, res))
    rec, paths = oracle_trace_sample(scene, cfg)
    from oracle import pathgraph_oracle as O

    n = rec["pos"].shape[0]
    for _ in range(args.warmup):
        g = O.build_graph(rec, paths, res, res, cfg.spp, cfg.cluster_size, cfg.seed)
        O.solve(g, cfg.iterations, 0.0)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        g = O.build_graph(rec, paths, res, res, cfg.spp, cfg.cluster_size, cfg.seed)
        O.solve(g, cfg.iterations, 0.0)
    dt = (time.perf_counter() - t0) / args.steps
    value = n / dt
    sample = (f"{wl.name} scene at {res}x{res}, {cfg.spp} spp ({n} vertices, traced by "
              f"oracle/tracer_oracle.c); build + {cfg.iterations} iterations per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": wl.name, "sample": f"{res}x{res}",
                                        "cluster_size": cfg.cluster_size,
                                        "iterations": cfg.iterations},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- native arm
def run_native(args):
    import torch

    from paper_2404_11894_b200 import _native as N
    from paper_2404_11894_b200.pathgraph import build_graph, solve
    from paper_2404_11894_b200.pathgraph.pipeline import solve_from_records
    from paper_2404_11894_b200.pathgraph.solve import splat_output_device
    from paper_2404_11894_b200.transport import render_pt
    from paper_2404_11894_b200.transport.records import PathSoA, RecordSoA, TraceOutput

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl, cfg = workload_config(args.workload)
    # multi-GPU: each rank renders its own frame of the workload (seed = rank)
    cfg.seed = rank
    scene = wl.scene()
    stream = torch.cuda.current_stream()

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    # ---- trace (setup; timed separately for ms/frame)
    trace = render_pt(scene, cfg, with_records=True)
    torch.cuda.synchronize()
    e0 = ev()
    trace = render_pt(scene, cfg, with_records=True)
    e1 = ev()
    torch.cuda.synchronize()
    trace_ms = e0.elapsed_time(e1)
    n = trace.records.n

    def step():
        g = build_graph(trace, cfg.cluster_size, seed=cfg.seed)
        res = solve(g, iterations=cfg.iterations, tol=0.0)
        return g, res

    for _ in range(args.warmup):
        g, res = step()
    del g, res
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches0 = N.launch_count()
    with ClockSampler(local) as clocks:
        time.sleep(0.25)  # let the sampler start before the timed region
        torch.cuda.synchronize()
        t_start = ev()
        for _ in range(args.steps):
            g, res = step()
        t_end = ev()
        torch.cuda.synchronize()
    launches = N.launch_count() - launches0
    step_ms = t_start.elapsed_time(t_end) / args.steps
    if dist:
        t = torch.tensor([step_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms = float(t.item())
    gi = g.info()

    # ---- splat (for ms/frame)
    s0 = ev()
    splat_output_device(g, res)
    s1 = ev()
    torch.cuda.synchronize()
    splat_ms = s0.elapsed_time(s1)
    del g, res

    # ---- per-kernel device times (one profiled step, after the timed region)
    N.profile_reset()
    N.profile(True)
    g, res = step()
    torch.cuda.synchronize()
    prof = N.profile_read()
    N.profile(False)
    N.profile_reset()
    prof_total = sum(ms for _, ms in prof.values())
    hbm, peak_kind = peaks()
    it_name = "k_solve_iter"
    it_count, it_ms = prof.get(it_name, (0, 0.0))
    it_avg_ms = it_ms / max(it_count, 1)
    achieved = ITER_BYTES_PER_VERTEX * n / (it_avg_ms * 1e-3) / 1e9 if it_count else 0.0
    traffic = None
    prof_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof_path):
        try:
            traffic = json.load(open(prof_path)).get(args.workload, {}).get(it_name)
        except Exception:
            traffic = None
    del g, res

    # ---- end to end through the public API with host buffers
    host_rec = RecordSoA(**trace.records.host_arrays()).pin_memory()
    host_paths = PathSoA(**trace.paths.host_arrays()).pin_memory()
    h2d_bytes = sum(a.nbytes for a in host_rec.host_arrays().values()) + \
        sum(a.nbytes for a in host_paths.host_arrays().values())

    def e2e_once():
        t = TraceOutput(None, RecordSoA(**host_rec.host_arrays()),
                        PathSoA(**host_paths.host_arrays()), trace.width, trace.height, trace.spp)
        t.records._pinned = host_rec._pinned
        t.paths._pinned = host_paths._pinned
        img, g2, r2 = solve_from_records(t, cfg.cluster_size, iterations=cfg.iterations, tol=0.0,
                                         seed=cfg.seed)
        return img

    e2e_once()
    torch.cuda.synchronize()
    tr0 = N.transfer_bytes()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        img = e2e_once()
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    tr1 = N.transfer_bytes()
    lib_h2d = (tr1[0] - tr0[0]) // args.e2e_steps
    lib_d2h = (tr1[1] - tr0[1]) // args.e2e_steps
    e2e = {"value": n * world / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": int(h2d_bytes + lib_h2d),
           "d2h_bytes_per_step": int(img.nbytes + lib_d2h),
           "ms_per_step": e2e_s * 1e3,
           "path": "pathgraph.pipeline.solve_from_records(host pinned records) -> image (host)"}

    # ---- CPU baseline (rank 0, N = 1 only): the oracle on a bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu, _, _ = cpu_baseline(wl, cfg, args.cpu_sample, device_trace_sample)
        except Exception as exc:  # never lose the GPU line over the baseline
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "port",
                   "sample": f"failed: {exc!r}"}

    value = n * world / (step_ms * 1e-3)
    step_bytes = (BUILD_BYTES_PER_VERTEX + ITER_BYTES_PER_VERTEX * cfg.iterations) * n
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (procedural fbm cloud scene, traced on device; no dataset)",
        "config": {"workload": wl.name, "resolution": list(wl.res), "spp": wl.spp,
                   "max_depth": wl.max_depth, "cluster_size": cfg.cluster_size,
                   "iterations": cfg.iterations, "tol": 0.0, "vertices_per_gpu": n,
                   "clusters": int(gi["n_clusters"]), "nnz": int(gi["nnz"]),
                   "parallelism": "replicas" if world > 1 else "single",
                   "l2": "inputs larger than L2 (records 290 B/vertex, kernel blocks 4 B/nnz)"},
        "ms_per_frame": trace_ms + step_ms + splat_ms,
        "frame_breakdown_ms": {"trace": trace_ms, "build_plus_solve": step_ms, "splat": splat_ms},
        "roofline": {"kernel": it_name, "bound": "hbm", "achieved": achieved, "peak": hbm,
                     "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                     "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": ITER_BYTES_PER_VERTEX * n,
                     "avg_launch_ms": it_avg_ms,
                     "share_of_step": it_ms / prof_total if prof_total else None},
        "step_roofline": {"algorithmic_bytes_per_step": step_bytes,
                          "achieved_gbs": step_bytes / (step_ms * 1e-3) / 1e9,
                          "frac": step_bytes / (step_ms * 1e-3) / 1e9 / hbm},
        "kernel_ms": {k: {"launches": c, "total_ms": ms} for k, (c, ms) in
                      sorted(prof.items(), key=lambda kv: -kv[1][1])},
        "build_stages": {"n_splits": int(gi["n_splits"]), "n_fallback": int(gi["n_fallback"])},
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_native(args)


if __name__ == "__main__":
    main()

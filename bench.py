#!/usr/bin/env python
"""Benchmark: graph vertices propagated/s (build + K iterations) and ms/frame.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]
                    [--workload C4] [--cpu-sample 64]

One step = one pass of the hot path over the workload's record set already
resident in HBM: build_graph (exact clustering, marginals, operator blocks)
+ solve(iterations=K_iter, tol=0).  `value` = vertices * N / step time.
`e2e` = the same metric through the reference-facing API with HOST buffers
(solve_from_records on pinned host records: H2D, build, solve, splat, image
D2H inside the timed region).  The workload is C4 (BASELINE.json configs[3]:
512^3 fbm smoke, 1024x1024, 16 spp, 16 iterations, ~75 M vertices), the
largest configuration that fits one GPU; it is traced by the CUDA tracer once,
outside the timed region; the synthetic smoke is procedural (no dataset).
Inputs (22 GB of records) are far larger than the 126 MB L2.

--impl reference times the reference algorithm's CPU restatement (oracle/,
numpy, with the reference's own control structure: per-cell candidate loop,
one nonzero() per center) on a bounded sample of the same workload (the C4
scene at 64x64, 16 spp) traced by the oracle's C tracer restatement, on the
host cores.
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
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--cpu-sample", type=int, default=64,
                    help="square resolution of the CPU-baseline sample of the workload")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-traffic", action="store_true",
                    help="skip the in-run ncu measurement of the roofline kernel's DRAM bytes")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--sharded", action="store_true",
                    help="run the row-partitioned multi-GPU path even at N=1 (default for N>1)")
    ap.add_argument("--no-sharded-n1", action="store_true",
                    help="skip the N=1 measurement of the sharded path beside the native one")
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
            # nvidia-smi's start-up (driver attach) must not fall into the
            # timed region: wait for its first sample
            t0 = time.time()
            while not self.rows and time.time() - t0 < 10.0 and self.proc.poll() is None:
                time.sleep(0.01)
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
        g = O.build_graph(rec, paths, sample_res, sample_res, cfg.spp, cfg.cluster_size, cfg.seed,
                          faithful=True)
        O.solve(g, cfg.iterations, 0.0)
        times.append(time.perf_counter() - t0)
    t = min(times)
    return {"value": n / t, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{wl.name} scene at {sample_res}x{sample_res}, {cfg.spp} spp: {n} vertices, "
                      f"build + {cfg.iterations} iterations in {t:.2f} s (oracle/pathgraph_oracle.py, "
                      f"numpy, the reference's per-cell / per-center loops, best of {steps}; "
                      f"single-threaded like the reference's graph stages)"}, n, t


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
    def step():
        g = O.build_graph(rec, paths, res, res, cfg.spp, cfg.cluster_size, cfg.seed, faithful=True)
        O.solve(g, cfg.iterations, 0.0)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    value = n / dt
    sample = (f"{wl.name} scene at {res}x{res}, {cfg.spp} spp ({n} vertices, traced by "
              f"oracle/tracer_oracle.c); build + {cfg.iterations} iterations per step "
              f"(numpy restatement with the reference's per-cell / per-center loops; "
              f"single-threaded like the reference's graph stages)")
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
    # the roofline kernel's DRAM traffic, measured in this run: ncu on a child
    # process that traces, builds and iterates the same workload, launched
    # first so that it has the GPU's memory to itself (nothing measured under
    # ncu is a bench value; the timed region comes later)
    measured_traffic = None
    if (not args.no_traffic and int(os.environ.get("WORLD_SIZE", "1")) == 1
            and args.gpus == 1):
        measured_traffic = ncu_traffic(args.workload, "k_solve_iter")
    import torch

    from paper_2404_11894_b200 import _native as N
    from paper_2404_11894_b200.pathgraph import build_graph, solve
    from paper_2404_11894_b200.pathgraph.pipeline import solve_from_records
    from paper_2404_11894_b200.pathgraph.solve import splat_output_device
    from paper_2404_11894_b200.transport import render_pt
    from paper_2404_11894_b200.transport import records as records_mod
    from paper_2404_11894_b200.transport.records import PathSoA, RecordSoA, TraceOutput

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl, cfg = workload_config(args.workload)
    scene = wl.scene()
    stream = torch.cuda.current_stream()

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    # ---- trace (setup; timed separately for ms/frame).  Each warm-up frame is
    # dropped before the next so the timed one reuses its memory, as a render
    # loop would.
    for _ in range(2):
        trace = render_pt(scene, cfg, with_records=True)
        del trace
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
        marks = []
        for _ in range(args.steps):
            g, res = step()
            marks.append(ev())
        t_end = marks[-1] if marks else ev()
        torch.cuda.synchronize()
    launches = N.launch_count() - launches0
    step_ms = t_start.elapsed_time(t_end) / args.steps
    each_ms = [round(a.elapsed_time(b), 3) for a, b in zip([t_start] + marks[:-1], marks)]
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
    traffic, traffic_source = None, None
    prof_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof_path):
        try:
            traffic = json.load(open(prof_path)).get(args.workload, {}).get(it_name)
            traffic_source = "profiles/traffic.json (ncu --set full of the same workload)"
        except Exception:
            traffic = None
    del g, res
    if measured_traffic:
        traffic, traffic_source = measured_traffic, (
            "ncu in this run (tools/traffic_probe.py, the third launch, before the timed region)")

    # ---- end to end through the public API with host buffers
    host_rec = RecordSoA(**trace.records.host_arrays()).pin_memory()
    host_paths = PathSoA(**trace.paths.host_arrays()).pin_memory()

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
    up0 = records_mod.h2d_bytes()  # record / path fields copied (only what the solve reads)
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        img = e2e_once()
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    tr1 = N.transfer_bytes()
    h2d_bytes = (records_mod.h2d_bytes() - up0) // args.e2e_steps
    lib_h2d = (tr1[0] - tr0[0]) // args.e2e_steps
    lib_d2h = (tr1[1] - tr0[1]) // args.e2e_steps
    e2e = {"value": n * world / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": int(h2d_bytes + lib_h2d),
           "d2h_bytes_per_step": int(img.nbytes + lib_d2h),
           "ms_per_step": e2e_s * 1e3,
           "path": "pathgraph.pipeline.solve_from_records(host pinned records) -> image (host)"}

    # ---- the N > 1 code path (pathgraph/sharded.py) at N = 1 on the same
    # records, so a scaling curve can be read against either N = 1 point
    sharded_n1 = None
    if world == 1 and not args.no_sharded_n1:
        try:
            sharded_n1 = sharded_step_n1(trace, cfg, args.steps, args.warmup, stream)
        except Exception as exc:  # never lose the GPU line over the side measurement
            sharded_n1 = {"error": repr(exc)}

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
        "warmup": args.warmup, "ms_per_step": step_ms, "step_ms_each": each_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (procedural fbm cloud scene, traced on device; no dataset)",
        "config": {"workload": wl.name, "resolution": list(wl.res), "spp": wl.spp,
                   "max_depth": wl.max_depth, "cluster_size": cfg.cluster_size,
                   "iterations": cfg.iterations, "tol": 0.0, "vertices_per_gpu": n,
                   "clusters": int(gi["n_clusters"]), "nnz": int(gi["nnz"]),
                   "parallelism": "single",
                   "l2": "inputs larger than L2 (records 290 B/vertex, kernel blocks 4 B/nnz)"},
        "ms_per_frame": trace_ms + step_ms + splat_ms,
        "frame_breakdown_ms": {"trace": trace_ms, "build_plus_solve": step_ms, "splat": splat_ms},
        "roofline": {"kernel": it_name, "bound": "hbm", "achieved": achieved, "peak": hbm,
                     "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                     # the block-dense layout moves fewer bytes than the CSR-based
                     # algorithmic figure (frac can exceed 1): the measured DRAM
                     # traffic over the same launch time is the hardware fraction
                     "traffic_gbs": (traffic / (it_avg_ms * 1e-3) / 1e9
                                     if traffic and it_count else None),
                     "traffic_frac": (traffic / (it_avg_ms * 1e-3) / 1e9 / hbm
                                      if traffic and it_count else None),
                     "traffic_source": traffic_source,
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
        "sharded_n1": sharded_n1,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def sharded_step_n1(trace, cfg, steps, warmup, stream):
    """The sharded path's build + solve (what bench.py runs for N > 1) on one
    GPU over the same device records: ms/step and vertices/s."""
    import torch

    from paper_2404_11894_b200.pathgraph.sharded import ShardComm, ShardedPathGraph

    from paper_2404_11894_b200 import _native as N

    N.release_cached()  # the native build's scratch / pool memory back for torch
    comm = ShardComm()
    recs = trace.records.device_tensors()
    n = trace.records.n

    def step():
        g = ShardedPathGraph.build(comm, recs, n, cfg.cluster_size, seed=cfg.seed)
        g.solve(cfg.iterations, 0.0)
        return g

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return {"value": n / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "steps": steps,
            "warmup": warmup,
            "path": "pathgraph/sharded.py ShardedPathGraph.build + solve at world 1 "
                    "(the code path of the N > 1 runs)"}


# ------------------------------------------------------------- sharded arm
def run_sharded(args):
    """N>1: one frame row-partitioned over the GPUs (pathgraph/sharded.py).

    Weak scaling: the frame is the workload at spp x N, so every GPU traces
    and owns about one C2 frame of records.  A step = the sharded build
    (light all-gather, exact clustering, record all-to-all, shard-local
    operators) + the solve with its per-iteration halo exchange.
    """
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2404_11894_b200 import _native as N
    from paper_2404_11894_b200.pathgraph.sharded import (ShardComm, ShardedPathGraph,
                                                         pixel_ranges)
    from paper_2404_11894_b200.scenecore.flatten import pack_scene
    from paper_2404_11894_b200.transport.tracer import trace_records_device

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = ShardComm()
    wl, cfg = workload_config(args.workload)
    cfg.spp = wl.spp * world
    scene = wl.scene()
    packed = pack_scene(scene)
    w, h, spp = packed.width, packed.height, cfg.spp
    ranges = pixel_ranges(w * h, world)
    p0, p1 = ranges[rank]
    stream = torch.cuda.current_stream()

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_ms(ms):
        t = torch.tensor([ms], device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    trace_records_device(scene, cfg, (p0 * spp, (p1 - p0) * spp))
    barrier()
    e0 = ev()
    recs, paths, n_rec = trace_records_device(scene, cfg, (p0 * spp, (p1 - p0) * spp))
    e1 = ev()
    barrier()
    trace_ms = max_ms(e0.elapsed_time(e1))

    def step():
        g = ShardedPathGraph.build(comm, recs, n_rec, cfg.cluster_size, seed=cfg.seed)
        g.pix_ranges = ranges
        g.solve(cfg.iterations, 0.0)
        return g

    for _ in range(args.warmup):
        g = step()
    del g
    barrier()
    launches0 = N.launch_count()
    with ClockSampler(local) as clocks:
        time.sleep(0.25)
        barrier()
        t_start = ev()
        for _ in range(args.steps):
            g = step()
        t_end = ev()
        barrier()
    launches = N.launch_count() - launches0
    step_ms = max_ms(t_start.elapsed_time(t_end) / args.steps)
    n_total = int(g.row_off[-1])
    n_own, n_halo = g.n, g.halo.n_halo
    s0 = ev()
    g.splat(paths, recs, (p0, p1), w, h, spp)
    s1 = ev()
    barrier()
    splat_ms = max_ms(s0.elapsed_time(s1))
    del g

    # per-kernel device times of one step (after the timed region)
    N.profile_reset()
    N.profile(True)
    g = step()
    barrier()
    prof = N.profile_read()
    N.profile(False)
    N.profile_reset()
    hbm, peak_kind = peaks()
    it_count, it_ms = prof.get("k_solve_iter", (0, 0.0))
    it_avg = it_ms / max(it_count, 1)
    achieved = ITER_BYTES_PER_VERTEX * g.n / (it_avg * 1e-3) / 1e9 if it_count else 0.0
    prof_total = sum(ms for _, ms in prof.values())
    del g

    # end to end: this shard's records from pinned host memory, image to the host
    host_recs = {k: v.cpu().pin_memory() for k, v in recs.items()}
    host_paths = {k: v.cpu().pin_memory() for k, v in paths.items()}
    h2d = sum(t.numel() * t.element_size() for t in list(host_recs.values()) +
              list(host_paths.values()))

    def e2e_once():
        r = {k: v.to("cuda", non_blocking=True) for k, v in host_recs.items()}
        pt = {k: v.to("cuda", non_blocking=True) for k, v in host_paths.items()}
        g2 = ShardedPathGraph.build(comm, r, n_rec, cfg.cluster_size, seed=cfg.seed)
        g2.pix_ranges = ranges
        g2.solve(cfg.iterations, 0.0)
        return g2.splat(pt, r, (p0, p1), w, h, spp).cpu()

    e2e_once()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        img = e2e_once()
    barrier()
    e2e_s = max_ms((time.perf_counter() - t0) / args.e2e_steps * 1e3) / 1e3

    value = n_total / (step_ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (procedural fbm cloud scene, traced on device; no dataset)",
        "config": {"workload": wl.name, "resolution": list(wl.res), "spp": spp,
                   "max_depth": wl.max_depth, "cluster_size": cfg.cluster_size,
                   "iterations": cfg.iterations, "tol": 0.0, "vertices_total": n_total,
                   "vertices_per_gpu": n_total / world, "rows_owned_rank0": n_own,
                   "halo_rows_rank0": n_halo, "parallelism": f"sharded{world}",
                   "frame": f"{wl.name} scene at {w}x{h}, spp = {wl.spp} x {world} GPUs",
                   "l2": "inputs larger than L2"},
        "ms_per_frame": trace_ms + step_ms + splat_ms,
        "frame_breakdown_ms": {"trace": trace_ms, "build_plus_solve": step_ms,
                               "splat": splat_ms},
        "roofline": {"kernel": "k_solve_iter", "bound": "hbm", "achieved": achieved,
                     "peak": hbm, "unit": "GB/s", "frac": achieved / hbm, "traffic": None,
                     "peak_kind": peak_kind, "avg_launch_ms": it_avg,
                     "share_of_step": it_ms / prof_total if prof_total else None},
        "kernel_ms": {k: {"launches": c, "total_ms": ms} for k, (c, ms) in
                      sorted(prof.items(), key=lambda kv: -kv[1][1])[:12]},
        "e2e": {"value": n_total / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(img.numel() * img.element_size()),
                "ms_per_step": e2e_s * 1e3,
                "path": "sharded build/solve/splat from pinned host records of each shard"},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
        "cpu_baseline": None,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def ncu_traffic(workload, kernel, timeout=420):
    """dram__bytes_read + dram__bytes_write of one steady-state launch of
    `kernel`, from ncu on tools/traffic_probe.py; None when ncu is missing or
    fails (the committed profiles/traffic.json figure is reported instead)."""
    import shutil
    import subprocess

    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--clock-control",
           "none", "-k", f"regex:{kernel}", "--launch-skip", "2", "--launch-count", "1", "--csv",
           sys.executable, os.path.join(ROOT, "tools", "traffic_probe.py"), workload]
    try:
        out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout).stdout
    except Exception:
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    total, seen = 0.0, 0
    import csv
    import io

    rows = [r for r in csv.reader(io.StringIO(out)) if len(r) > 3]
    if not rows:
        return None
    hdr = rows[0]
    if "Metric Name" not in hdr:
        return None
    mi, ui, vi = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    for r in rows[1:]:
        if r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            try:
                total += float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
                seen += 1
            except ValueError:
                pass
    return int(total) if seen == 2 else None


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.sharded or dist_env()[1] > 1:
        run_sharded(args)
    else:
        run_native(args)


if __name__ == "__main__":
    main()

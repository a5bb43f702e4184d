"""Row-partitioned path graph: one shard per GPU (option B).

The reference is single-process (pipeline.py:25-42); this module spreads one
frame over the processes of a torch.distributed group, one per GPU, and gives
bit-identical results to the single-GPU path for any shard count:

  trace    each shard traces a contiguous, pixel-aligned range of camera
           paths.  Path ids and their splitmix64 streams are global
           (tracer.py:58-70, rng.py:19-45), so the shards' records, in
           shard order, are exactly the single-GPU record set.
  cluster  the light columns (pos, kind, class_id: 29 B/record) are
           all-gathered and every shard runs the exact clustering
           (clustering.py:28-148) on the whole set; same input and
           deterministic code give the same clusters on every shard.
  own      clusters are ordered by the Morton code of their center and cut
           into contiguous ranges of equal solve cost (sum of s^2 + 16 s
           floats), one per shard; every record moves once, in one
           all-to-all, to the shard that owns its cluster, laid out
           cluster-major with members in ascending record order.
  build    each shard builds the marginals, kernel blocks and D-bar of its
           own clusters (vpg_graph_build_local, graph.py:94-168) — the same
           arithmetic on the same members as the single-GPU build.
  solve    per iteration (solve.py:78-94) rows whose continuation parent
           lives on another shard write into halo slots, one all-to-all
           delivers them to the parent's shard, and the 7 residual words are
           max-reduced, so every shard takes the same tol / divergence
           decision.  This is the path's only per-iteration exchange:
           f_cross x 16 B per row instead of an all-gather of I.
  splat    the owners of the paths' first records send (W I, D-bar) back to
           the path shards, which splat their pixel ranges (solve.py:101-132);
           the image is all-gathered.

Collectives go through torch.distributed: NCCL on device memory in
production, gloo (through host memory) for the CPU-side tests and for
several shards sharing one GPU in the parity test.  No kernel waits on
another shard: exchanges happen between launches.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from paper_2404_11894_b200 import _native as N
from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.scenecore.flatten import pack_scene

_FLOAT_WORDS = 6   # residual maxima per iteration (solve.py:54-61)
_NAN_WORD = 6      # per-channel NaN flags


# --------------------------------------------------------------- collectives
class ShardComm:
    """The collectives of the sharded path over a torch.distributed group.

    NCCL exchanges device tensors directly; any other backend (gloo) stages
    through host memory.  With one process (or no initialised group) every
    call is a local no-op, so the same code runs a single shard.
    """

    def __init__(self, group=None):
        import torch.distributed as dist

        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.dist = dist
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
            self.backend = str(dist.get_backend(group))
        else:
            self.dist, self.rank, self.world, self.backend = None, 0, 1, "none"
        self.staged = self.backend != "nccl"

    def _out(self, t):
        return t.cpu() if self.staged else t

    def all_to_all(self, send, send_counts, recv_counts):
        """Rows of `send` grouped by destination shard -> rows received, grouped by source."""
        import torch

        send_counts = [int(c) for c in send_counts]
        recv_counts = [int(c) for c in recv_counts]
        if self.world == 1:
            return send.clone()
        src = self._out(send.contiguous())
        out = torch.empty((sum(recv_counts),) + tuple(send.shape[1:]), dtype=send.dtype,
                          device=src.device)
        self.dist.all_to_all_single(out, src, recv_counts, send_counts, group=self.group)
        return out.to(send.device)

    def all_gather_rows(self, t, counts):
        """Concatenate every shard's rows (shard r contributes counts[r] rows)."""
        import torch

        counts = [int(c) for c in counts]
        if self.world == 1:
            return t.clone()
        mx = max(max(counts), 1)
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        pad = self._out(pad)
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(parts, pad, group=self.group)
        return torch.cat([p[:c] for p, c in zip(parts, counts)]).to(t.device)

    def all_gather_ints(self, values):
        """Every shard's list of ints -> (world, len) int64 numpy array."""
        import torch

        v = torch.tensor([int(x) for x in values], dtype=torch.int64)
        if self.world == 1:
            return v.numpy()[None, :]
        dev = "cpu" if self.staged else "cuda"
        v = v.to(dev)
        parts = [torch.empty_like(v) for _ in range(self.world)]
        self.dist.all_gather(parts, v, group=self.group)
        return torch.stack(parts).cpu().numpy()

    def all_reduce_max_(self, t):
        """In-place elementwise max over the shards."""
        if self.world == 1:
            return t
        src = self._out(t)
        self.dist.all_reduce(src, op=self.dist.ReduceOp.MAX, group=self.group)
        if src is not t:
            t.copy_(src)
        return t


# --------------------------------------------------------------- device views
class _CAI:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


def _view(ptr, shape, typestr):
    """A torch tensor aliasing device memory owned by the native graph."""
    import torch

    if not ptr or int(np.prod(shape)) == 0:
        dt = {"<f4": torch.float32, "<i4": torch.int32}[typestr]
        return torch.empty(shape, dtype=dt, device="cuda")
    return torch.as_tensor(_CAI(ptr, shape, typestr), device="cuda")


# ----------------------------------------------------------------- planning
def pixel_ranges(n_pix: int, world: int):
    """Contiguous, balanced pixel ranges; a pixel's samples stay on one shard so
    its spp mean is summed in sample order exactly as on one GPU."""
    return [(r * n_pix // world, (r + 1) * n_pix // world) for r in range(world)]


def morton3(q):
    """Interleave the low 21 bits of the three int64 columns of q (z-order)."""
    def spread(v):
        v = v & 0x1FFFFF
        v = (v | (v << 32)) & 0x1F00000000FFFF
        v = (v | (v << 16)) & 0x1F0000FF0000FF
        v = (v | (v << 8)) & 0x100F00F00F00F00F
        v = (v | (v << 4)) & 0x10C30C30C30C30C3
        v = (v | (v << 2)) & 0x1249249249249249
        return v
    return spread(q[:, 0]) | (spread(q[:, 1]) << 1) | (spread(q[:, 2]) << 2)


@dataclass
class OwnerPlan:
    owner: "object"        # (M,) int64 shard of each cluster (clustering's internal order)
    order: "object"        # (M,) clusters in Morton order (ranges of it are the shards)
    local_start: "object"  # (M,) first row of the cluster in its owner's layout
    rows: list             # rows owned per shard
    clusters: list         # clusters owned per shard


def plan_owners(cl_size, center_pos, world: int) -> OwnerPlan:
    """Morton-ordered clusters cut into `world` contiguous ranges of equal cost."""
    import torch

    m = int(cl_size.shape[0])
    dev = cl_size.device
    size = cl_size.to(torch.int64)
    if m == 0:
        z = torch.zeros(0, dtype=torch.int64, device=dev)
        return OwnerPlan(z, z, z, [0] * world, [0] * world)
    lo = center_pos.min(0).values
    ext = (center_pos.max(0).values - lo).clamp_min(1e-300)
    q = ((center_pos - lo) / ext * 2097151.0).floor().clamp(0, 2097151).to(torch.int64)
    order = torch.argsort(morton3(q), stable=True)
    cost = size[order] * size[order] + 16 * size[order]
    before = torch.cumsum(cost, 0) - cost
    total = int(cost.sum())
    own_o = torch.clamp((2 * before + cost) * world // max(2 * total, 1), max=world - 1)
    owner = torch.empty(m, dtype=torch.int64, device=dev)
    owner[order] = own_o
    s_o = size[order]
    excl = torch.cumsum(s_o, 0) - s_o
    first_row = torch.zeros(world, dtype=torch.int64, device=dev)
    rows_per = torch.zeros(world, dtype=torch.int64, device=dev).index_add_(0, own_o, s_o)
    first_row[1:] = torch.cumsum(rows_per, 0)[:-1]
    local_start = torch.empty(m, dtype=torch.int64, device=dev)
    local_start[order] = excl - first_row[own_o]
    clusters_per = torch.bincount(own_o, minlength=world)
    return OwnerPlan(owner, order, local_start, [int(x) for x in rows_per.tolist()],
                     [int(x) for x in clusters_per.tolist()])


def row_destinations(perm, cl_off, plan: OwnerPlan):
    """(dest_shard, dest_row) of every record (global record order)."""
    import torch

    n = int(perm.shape[0])
    m = int(cl_off.shape[0]) - 1
    dev = perm.device
    off = cl_off.to(torch.int64)
    sizes = off[1:] - off[:-1]
    k_of_q = torch.repeat_interleave(torch.arange(m, device=dev), sizes)
    within = torch.arange(n, device=dev) - off[k_of_q]
    rec = perm.to(torch.int64)
    dest_shard = torch.empty(n, dtype=torch.int64, device=dev)
    dest_row = torch.empty(n, dtype=torch.int64, device=dev)
    dest_shard[rec] = plan.owner[k_of_q]
    dest_row[rec] = plan.local_start[k_of_q] + within
    return dest_shard, dest_row


def recv_counts_for(dest_shard, row_counts, me: int, world: int):
    """Rows shard `me` receives from each source shard (rows are in shard order)."""
    import torch

    src = torch.repeat_interleave(torch.arange(world, device=dest_shard.device),
                                  torch.as_tensor(row_counts, device=dest_shard.device))
    return torch.bincount(src[dest_shard == me], minlength=world).tolist()


class HaloExchange:
    """Continuation edges that cross shards (solve.py:78-83 propagation).

    Local rows whose parent record lives on another shard propagate into halo
    slots n .. n + n_halo - 1, ordered by (parent shard, parent row); after
    every iteration one all-to-all delivers the slots to the parents' shards,
    which write them into their rows."""

    def __init__(self, comm: ShardComm, n_local: int, parent_shard, parent_row, child_rows):
        import torch

        self.comm = comm
        self.n = n_local
        key = parent_shard * 2 ** 32 + parent_row  # (shard, row) lexicographic; rows < 2^31
        srt = torch.argsort(key, stable=True)
        self.child_rows = child_rows[srt]
        self.n_halo = int(srt.numel())
        dst = parent_shard[srt]
        self.send_counts = torch.bincount(dst, minlength=comm.world).tolist() \
            if self.n_halo else [0] * comm.world
        counts = torch.tensor(self.send_counts, dtype=torch.int64, device=parent_row.device)
        recv = comm.all_to_all(counts.reshape(-1, 1), [1] * comm.world, [1] * comm.world)
        self.recv_counts = recv.reshape(-1).tolist()
        self.recv_rows = comm.all_to_all(parent_row[srt], self.send_counts, self.recv_counts)

    def exchange(self, i_out):
        """i_out: (n + n_halo, C) — send the halo rows, write the received ones."""
        if self.comm.world == 1:
            return
        got = self.comm.all_to_all(i_out[self.n:self.n + self.n_halo], self.send_counts,
                                   self.recv_counts)
        if got.shape[0]:
            i_out[self.recv_rows] = got


# ------------------------------------------------------------ record payload
def _payload_columns():
    cols = []
    for name, width, code in N.RECORD_FIELDS:
        cols.append((name, width, code))
    cols += [("parent_ipt", 3, "f8"), ("has_child", 1, "i8"), ("grow", 1, "i8"),
             ("dest_row", 1, "i8")]
    return cols


def _torch_dtype(code):
    import torch

    return {"f8": torch.float64, "i8": torch.int64, "i4": torch.int32, "u1": torch.uint8}[code]


def pack_payload(cols: dict, n: int):
    """Record columns -> (n, W) float64, integer columns bit-cast (exact transport)."""
    import torch

    parts = []
    for name, width, code in _payload_columns():
        t = cols[name].reshape(n, width)
        if code == "f8":
            parts.append(t)
        else:
            parts.append(t.to(torch.int64).view(torch.float64))
    return torch.cat(parts, 1) if parts else None


def unpack_payload(p):
    import torch

    out, c = {}, 0
    for name, width, code in _payload_columns():
        t = p[:, c:c + width]
        c += width
        if code != "f8":
            t = t.contiguous().view(torch.int64).to(_torch_dtype(code))
        t = t.contiguous()
        out[name] = t if width > 1 else t.reshape(-1)
    return out


# ------------------------------------------------------------- the shard
@dataclass
class ShardedSolve:
    residuals: list
    iterations: int


class ShardedPathGraph:
    """This shard's part of the path graph (its clusters' rows + halo)."""

    def __init__(self):
        self.handle = None

    def __del__(self):
        if getattr(self, "handle", None):
            try:
                N.lib().vpg_graph_free(self.handle)
            except Exception:
                pass
            self.handle = None

    # -- build ---------------------------------------------------------------
    @classmethod
    def build(cls, comm: ShardComm, recs: dict, n_rec: int, cluster_size: int, seed: int = 0):
        """recs: this shard's trace records (device tensors, path order)."""
        import torch

        if cluster_size < 1:
            raise ValueError("cluster size K must be >= 1")
        self = cls()
        self.comm = comm
        me, world = comm.rank, comm.world
        stream = N.stream_handle()
        lib = N.lib()
        counts = comm.all_gather_ints([n_rec])[:, 0].tolist()
        self.row_counts = counts
        self.row_off = [0] + list(np.cumsum(counts))
        n_all = int(self.row_off[-1])
        # light columns of every record, then the exact clustering on all of them
        pos = comm.all_gather_rows(recs["pos"][:n_rec], counts)
        kind = comm.all_gather_rows(recs["kind"][:n_rec], counts)
        cls_id = comm.all_gather_rows(recs["class_id"][:n_rec], counts)
        light = N.Records()
        light.n = n_all
        if n_all:
            light.pos, light.kind, light.class_id = pos.data_ptr(), kind.data_ptr(), cls_id.data_ptr()
        rng = np.random.default_rng(np.random.SeedSequence([seed & 0xFFFFFFFF, 0xC1A5]))
        st = N.Pcg64State.from_generator(rng)
        gc = ctypes.c_void_p()
        N.check(lib.vpg_graph_build(ctypes.byref(light), int(cluster_size), ctypes.byref(st),
                                    N.VPG_BUILD_CLUSTERS_ONLY, stream, ctypes.byref(gc)))
        try:
            v = N.GraphViews()
            N.check(lib.vpg_graph_views_get(gc.value, ctypes.byref(v)))
            m = int(v.m)
            perm = _view(v.perm, (n_all,), "<i4").clone()
            cl_off = _view(v.cl_off, (m + 1,), "<i4").clone()
            center = _view(v.cl_center, (m,), "<i4").clone()
        finally:
            lib.vpg_graph_free(gc.value)
        self.n_clusters_total = m
        sizes = (cl_off[1:] - cl_off[:-1]).to(torch.int64)
        plan = plan_owners(sizes, pos[center.to(torch.int64)] if m else pos[:0], world)
        dest_shard, dest_row = row_destinations(perm, cl_off, plan)
        self.plan = plan
        del pos, kind, cls_id, perm

        # this shard's records, with what the owner needs beyond them
        n = n_rec
        g0 = int(self.row_off[me])
        cols = {name: recs[name][:n] for name, _, _ in N.RECORD_FIELDS}
        pidx = cols["path_idx"]
        has_child = torch.zeros(n, dtype=torch.int64, device="cuda")
        if n > 1:
            has_child[:-1] = (pidx[1:] == pidx[:-1]).to(torch.int64)
        parent_ipt = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
        if n > 1:
            parent_ipt[1:] = cols["i_pt"][:-1]
        parent_ipt[cols["depth"] == 0] = 0.0
        grow = torch.arange(g0, g0 + n, dtype=torch.int64, device="cuda")
        cols.update(parent_ipt=parent_ipt, has_child=has_child, grow=grow,
                    dest_row=dest_row[g0:g0 + n])
        dst = dest_shard[g0:g0 + n]
        order = torch.argsort(dst, stable=True)
        send_counts = torch.bincount(dst, minlength=world).tolist() if n else [0] * world
        recv_counts = recv_counts_for(dest_shard, counts, me, world)
        payload = pack_payload(cols, n)
        got = comm.all_to_all(payload[order], send_counts, recv_counts)
        n_own = int(plan.rows[me])
        local = torch.empty((n_own, got.shape[1]), dtype=torch.float64, device="cuda")
        rows_at = got[:, -1].contiguous().view(torch.int64)
        local[rows_at] = got
        own = unpack_payload(local)
        self.own = own
        self.n = n_own

        # continuation parents: local row, or a halo slot for a remote one
        depth = own["depth"].to(torch.int64)
        has_par = depth > 0
        par_g = own["grow"] - 1
        parent = torch.full((n_own,), -1, dtype=torch.int64, device="cuda")
        rows_with = torch.nonzero(has_par).reshape(-1)
        p_shard = dest_shard[par_g[rows_with]]
        p_row = dest_row[par_g[rows_with]]
        local_mask = p_shard == me
        parent[rows_with[local_mask]] = p_row[local_mask]
        remote = ~local_mask
        self.halo = HaloExchange(comm, n_own, p_shard[remote], p_row[remote], rows_with[remote])
        parent[self.halo.child_rows] = n_own + torch.arange(self.halo.n_halo, device="cuda")
        halo_ipt = own["parent_ipt"][self.halo.child_rows].contiguous()
        self.parent = parent.to(torch.int32)
        self.has_child = own["has_child"].to(torch.uint8)
        self.halo_ipt = halo_ipt
        del dest_shard, dest_row

        # operators of this shard's clusters
        own_clusters = plan.order[plan.owner[plan.order] == me]
        cl_sizes = sizes[own_clusters].to(torch.int32).cpu().numpy()
        self.cl_sizes = cl_sizes
        st = N.Records()
        st.n = n_own
        for name, _, _ in N.RECORD_FIELDS:
            t = own[name]
            setattr(st, name, t.data_ptr() if t.numel() else None)
        self._rec_struct = st
        g = ctypes.c_void_p()
        N.check(lib.vpg_graph_build_local(
            ctypes.byref(st), int(cl_sizes.size), cl_sizes.ctypes.data if cl_sizes.size else None,
            self.parent.data_ptr() if n_own else None,
            self.has_child.data_ptr() if n_own else None, self.halo.n_halo,
            halo_ipt.data_ptr() if self.halo.n_halo else None, stream, ctypes.byref(g)))
        self.handle = g.value
        # the residual scale covers every shard's terminal rows (solve.py:57-60)
        vw = self.views()
        comm.all_reduce_max_(_view(vw.term_max, (3,), "<f4"))
        self.performed = -1
        return self

    def views(self):
        v = N.GraphViews()
        N.check(N.lib().vpg_graph_views_get(self.handle, ctypes.byref(v)))
        return v

    # -- solve ---------------------------------------------------------------
    def solve(self, iterations: int = 10, tol: float = 1e-3) -> ShardedSolve:
        import torch

        from paper_2404_11894_b200.pathgraph.solve import SolveDivergence

        if iterations < 0:
            raise ValueError("iterations must be >= 0")
        lib, stream = N.lib(), N.stream_handle()
        N.check(lib.vpg_solve_begin(self.handle, int(iterations), float(tol), stream))
        v = self.views()
        rows = self.n + self.halo.n_halo
        red_f = _view(v.red, ((iterations + 1) * 8,), "<f4")
        red_i = _view(v.red, ((iterations + 1) * 8,), "<i4")
        bit = torch.arange(6, device="cuda", dtype=torch.int32)
        for t in range(iterations):
            N.check(lib.vpg_solve_step(self.handle, t, stream))
            if self.comm.world > 1:
                i_out = _view(v.ibuf[(t + 1) & 1], (rows, 4), "<f4")
                self.halo.exchange(i_out)
                words = red_f[t * 8:t * 8 + _FLOAT_WORDS]
                self.comm.all_reduce_max_(words)
                nan = (red_i[t * 8 + _NAN_WORD] >> bit) & 1
                self.comm.all_reduce_max_(nan)
                red_i[t * 8 + _NAN_WORD] = (nan << bit).sum().to(torch.int32)
            N.check(lib.vpg_solve_control(self.handle, t, stream))
        res = np.zeros(max(iterations, 1))
        performed = ctypes.c_int32(0)
        rc = lib.vpg_solve_end(self.handle, res.ctypes.data, ctypes.byref(performed), stream)
        self.performed = performed.value
        residuals = [float(r) for r in res[:performed.value]]
        if rc == N.VPG_EDIVERGED:
            raise SolveDivergence("fixed-point residuals grew over 3 consecutive iterations "
                                  f"({residuals[-4:]})")
        N.check(rc)
        return ShardedSolve(residuals, performed.value)

    # -- results -------------------------------------------------------------
    def _acc(self):
        v = self.views()
        return (_view(v.acc[self.performed & 1], (self.n, 4), "<f4"),
                _view(v.dbar, (self.n, 4), "<f4"),
                _view(v.ibuf[self.performed & 1], (self.n + self.halo.n_halo, 4), "<f4"))

    def gather_solution(self):
        """(incoming, i_bar) of every record, global record order, float64 —
        the SolveResult fields (solve.py:28-34) on every shard."""
        import torch

        acc, _, ibuf = self._acc()
        incoming = ibuf[:self.n, :3].to(torch.float64)
        i_bar = self.own["coeff"] * acc[:, :3].to(torch.float64)
        counts = self.comm.all_gather_ints([self.n])[:, 0].tolist()
        rows = self.comm.all_gather_rows(self.own["grow"], counts)
        vals = self.comm.all_gather_rows(torch.cat([incoming, i_bar], 1), counts)
        out = torch.empty_like(vals)
        out[rows] = vals
        return out[:, :3], out[:, 3:]

    def splat(self, paths: dict, recs: dict, pix_range, width: int, height: int, spp: int,
              mode: int = N.DIRECT_PT):
        """splat_output (solve.py:101-132) of this shard's pixels; returns the
        full (H, W, 3) image on every shard."""
        import torch

        comm, me, world = self.comm, self.comm.rank, self.comm.world
        acc, dbar, _ = self._acc()
        first = torch.nonzero(self.own["depth"] == 0).reshape(-1)
        pid = self.own["path_idx"][first]
        starts = torch.tensor([r[0] * spp for r in self.pix_ranges] + [width * height * spp],
                              dtype=torch.int64, device="cuda")
        dst = torch.searchsorted(starts, pid, right=True) - 1
        order = torch.argsort(dst, stable=True)
        msg = torch.cat([acc[first], dbar[first],
                         (pid - starts[dst]).reshape(-1, 1).view(torch.float32).reshape(-1, 2)],
                        1)[order]
        send_counts = torch.bincount(dst, minlength=world).tolist() if first.numel() else \
            [0] * world
        cnt = comm.all_to_all(torch.tensor(send_counts, dtype=torch.int64,
                                           device="cuda").reshape(-1, 1), [1] * world, [1] * world)
        got = comm.all_to_all(msg.contiguous(), send_counts, cnt.reshape(-1).tolist())
        p0, p1 = pix_range
        n_paths = (p1 - p0) * spp
        acc_first = torch.zeros((n_paths + 1, 4), dtype=torch.float32, device="cuda")
        dbar_first = torch.zeros((n_paths + 1, 4), dtype=torch.float32, device="cuda")
        idx = got[:, 8:10].contiguous().view(torch.int64).reshape(-1)
        acc_first[idx] = got[:, 0:4]
        dbar_first[idx] = got[:, 4:8]
        n_loc = int(recs["pos"].shape[0])
        clpos = torch.zeros(max(n_loc, 1), dtype=torch.int32, device="cuda")
        has = paths["rec_count"] > 0
        clpos[paths["rec_start"][has]] = torch.nonzero(has).reshape(-1).to(torch.int32)
        pst = N.Paths()
        pst.n = n_paths
        for name, _, _ in N.PATH_FIELDS:
            t = paths[name]
            setattr(pst, name, t.data_ptr() if t.numel() else None)
        img = torch.zeros(((p1 - p0) + 1, 3), dtype=torch.float64, device="cuda")
        if p1 > p0:
            N.check(N.lib().vpg_splat_arrays(ctypes.byref(pst), recs["coeff"].data_ptr()
                                             if n_loc else None, clpos.data_ptr(),
                                             acc_first.data_ptr(), dbar_first.data_ptr(), p1 - p0,
                                             spp, int(mode), img.data_ptr(), N.stream_handle()))
        counts = [b - a for a, b in self.pix_ranges]
        full = comm.all_gather_rows(img[:p1 - p0], counts)
        return full.reshape(height, width, 3)


@dataclass
class ShardedRender:
    image: np.ndarray
    residuals: list
    iterations: int
    graph: ShardedPathGraph
    n_records: int        # this shard's traced records
    n_records_total: int


def render_pg_sharded(scene, config: RenderConfig, comm: ShardComm | None = None,
                      keep_graph: bool = True) -> ShardedRender:
    """render_pg (pipeline.py:25-42) over the shards of `comm` (default: the
    initialised torch.distributed group, or a single shard)."""
    from paper_2404_11894_b200.transport.tracer import trace_records_device

    comm = comm or ShardComm()
    if config.extra_direct_samples > 0:
        raise ValueError("extra_direct_samples is not supported on the sharded path")
    packed = pack_scene(scene)
    w, h, spp = packed.width, packed.height, int(config.spp)
    ranges = pixel_ranges(w * h, comm.world)
    p0, p1 = ranges[comm.rank]
    recs, paths, n_rec = trace_records_device(scene, config, ((p0 * spp), (p1 - p0) * spp))
    g = ShardedPathGraph.build(comm, recs, n_rec, config.cluster_size, seed=config.seed)
    g.pix_ranges = ranges
    sol = g.solve(config.iterations, config.tol)
    mode = N.DIRECT_AGGREGATED if config.aggregate_direct else N.DIRECT_PT
    img = g.splat(paths, recs, (p0, p1), w, h, spp, mode)
    total = int(g.row_off[-1])
    return ShardedRender(image=img.cpu().numpy(), residuals=sol.residuals,
                         iterations=sol.iterations, graph=g if keep_graph else None,
                         n_records=n_rec, n_records_total=total)

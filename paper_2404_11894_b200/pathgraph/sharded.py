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
           delivers them to the parent's shard, and the 6 residual words are
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
import os
from dataclasses import dataclass

import numpy as np

from paper_2404_11894_b200 import _native as N
from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.scenecore.flatten import pack_scene

_RESIDUAL_WORDS = 6  # residual maxima per iteration (solve.py:54-61), float bits


# --------------------------------------------------------------- collectives
class ShardComm:
    """The collectives of the sharded path over a torch.distributed group.

    NCCL exchanges device tensors directly; any other backend (gloo) stages
    through host memory.  With one process (or no initialised group) every
    call is a local no-op, so the same code runs a single shard --
    `loopback=True` sends them through the group anyway (a one-rank NCCL group
    then runs every NCCL call of the N > 1 path on one GPU).
    """

    def __init__(self, group=None, loopback=False):
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
        # skip the collectives only for a single rank that is not looped back
        self.local = self.world == 1 and not (loopback and self.dist is not None)

    def _out(self, t):
        return t.cpu() if self.staged else t

    def all_to_all(self, send, send_counts, recv_counts):
        """Rows of `send` grouped by destination shard -> rows received, grouped by source."""
        import torch

        send_counts = [int(c) for c in send_counts]
        recv_counts = [int(c) for c in recv_counts]
        if self.local:
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
        if self.local:
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
        if self.local:
            return v.numpy()[None, :]
        dev = "cpu" if self.staged else "cuda"
        v = v.to(dev)
        parts = [torch.empty_like(v) for _ in range(self.world)]
        self.dist.all_gather(parts, v, group=self.group)
        return torch.stack(parts).cpu().numpy()

    def exclusive_scan(self, v):
        """(sum of v over the shards before this one, sum over all shards) for
        an integer vector of equal length on every shard.  Shards own
        contiguous blocks of the vector: one all-to-all sends each block to its
        owner, which scans it across the shards and returns every shard its
        prefix and the total (3 m words moved per shard instead of the
        world * m of an all-gather)."""
        import torch

        m = int(v.shape[0])
        if self.local:
            return torch.zeros_like(v), v.clone()
        if self.world == 2:  # the all-gather is already as small
            rows = self.all_gather_rows(v.reshape(1, -1), [1, 1])
            return rows[: self.rank].sum(0), rows.sum(0)
        w = self.world
        cuts = [m * k // w for k in range(w + 1)]
        sizes = [cuts[k + 1] - cuts[k] for k in range(w)]
        # to owner k: my slice [cuts[k], cuts[k+1])
        got = self.all_to_all(v, sizes, [sizes[self.rank]] * w)
        mine = got.reshape(w, sizes[self.rank])
        total = mine.sum(0)
        before = torch.cumsum(mine, 0) - mine          # row r: sum over shards < r
        back = torch.cat([before, total.reshape(1, -1).expand(w, -1)], 1)  # (w, 2 * my size)
        ret = self.all_to_all(back.reshape(-1), [2 * sizes[self.rank]] * w,
                              [2 * sz for sz in sizes])
        pre, tot = [], []
        at = 0
        for sz in sizes:
            pre.append(ret[at:at + sz])
            tot.append(ret[at + sz:at + 2 * sz])
            at += 2 * sz
        return torch.cat(pre), torch.cat(tot)

    def all_reduce_max_(self, t):
        """In-place elementwise max over the shards."""
        if self.local:
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
        if self.comm.local:
            return
        got = self.comm.all_to_all(i_out[self.n:self.n + self.n_halo], self.send_counts,
                                   self.recv_counts)
        if got.shape[0]:
            i_out[self.recv_rows] = got


# ------------------------------------------------------ distributed clustering
def _sq_dist(a, b):
    """fp64 squared distance rounded like numpy's ((a-b)**2).sum(-1): ((dx*dx + dy*dy) + dz*dz),
    one IEEE op at a time (no contraction)."""
    d = a - b
    sq = d * d
    return (sq[:, 0] + sq[:, 1]) + sq[:, 2]


@dataclass
class GlobalClusters:
    """The clusters of the whole frame (replicated on every shard) and this
    shard's rows' places in them."""
    sizes: "object"       # (M,) int64, reference cluster order
    center_pos: "object"  # (M, 3) float64
    row_cluster: "object"  # (n_local,) int64
    row_rank: "object"     # (n_local,) int64 rank in the cluster (ascending global row)
    n_splits: int


_TIMING = os.environ.get("VPG_SHARD_TIMING") is not None
_T = {"t": 0.0}


def _tick(label):
    """VPG_SHARD_TIMING=1: print the wall time since the previous tick (synced)."""
    if not _TIMING:
        return
    import time

    import torch

    torch.cuda.synchronize()
    now = time.perf_counter()
    if _T["t"]:
        print(f"[shard] {label:28s} {1e3 * (now - _T['t']):8.3f} ms", flush=True)
    _T["t"] = now


def _local_class_keys(keys):
    """np.unique of this shard's class keys (kind << 32 | class_id), ascending:
    one min/max pass when every row has the same key (the usual single
    class), a presence map over the key range when it is small, else a sort."""
    import torch

    lo, hi = torch.aminmax(keys)
    lo, hi = int(lo), int(hi)
    if lo == hi:
        return keys[:1].clone()
    if hi - lo < 1 << 20:
        seen = torch.zeros(hi - lo + 1, dtype=torch.bool, device=keys.device)
        seen.index_fill_(0, keys - lo, True)
        return torch.nonzero(seen).reshape(-1) + lo
    return torch.unique(keys)


def cluster_distributed(comm: ShardComm, pos, kind, class_id, g0: int, cluster_size: int,
                        rng: np.random.Generator) -> GlobalClusters:
    """cluster_points (clustering.py:28-148) over the shards' records without
    gathering them: per class (ascending keys) the centers are drawn with the
    replicated Generator (numpy's own choice, the same stream on every
    shard), their positions all-gathered from the shards holding them, every
    shard assigns its own rows (exact nearest, lowest index on ties), the
    group sizes are all-reduced, and only the oversize groups' members are
    gathered for the split loop, which runs replicated on the shared stream.
    Same clusters as the single-device build."""
    import torch

    dev = pos.device
    me, world = comm.rank, comm.world
    K = int(cluster_size)
    max_size = 2 * K
    n = int(pos.shape[0])
    _tick("cd: start")
    keys = (kind.to(torch.int64) << 32) | class_id.to(torch.int64)
    loc_keys = _local_class_keys(keys) if n else keys[:0]
    cnt = comm.all_gather_ints([int(loc_keys.numel())])[:, 0].tolist()
    all_keys = comm.all_gather_rows(loc_keys, cnt)
    classes = sorted(set(int(x) for x in all_keys.cpu().tolist()))
    sizes_all, cpos_all = [], []
    row_cluster = torch.full((n,), -1, dtype=torch.int64, device=dev)
    row_rank = torch.full((n,), -1, dtype=torch.int64, device=dev)
    base = 0
    n_splits = 0
    lib = N.lib()
    stream = N.stream_handle()
    for key in classes:
        if len(classes) == 1:  # every row (no class filter, no copy of pos)
            rows = torch.arange(n, device=dev)
        else:
            rows = torch.nonzero(keys == key).reshape(-1)  # ascending = ascending global row
        counts = comm.all_gather_ints([int(rows.numel())])[:, 0]
        n_c = int(counts.sum())
        pref = int(counts[:me].sum())
        my_n = int(rows.numel())
        m = -(-n_c // K)
        # centers: Generator.choice(n, m, replace=False) (clustering.py:51), by
        # the native bit-exact replica (host draws, swaps resolved on the device)
        _tick("cd: class rows")
        idx32 = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
        st0 = N.Pcg64State.from_generator(rng)
        N.check(lib.vpg_rng_choice_device(ctypes.byref(st0), n_c, m, idx32.data_ptr(), stream))
        st0.store_into(rng)
        idx = idx32[:m].to(torch.int64)
        mine = torch.nonzero((idx >= pref) & (idx < pref + my_n)).reshape(-1)
        c_rows = rows[idx[mine] - pref]
        msg = torch.cat([mine.to(torch.float64).reshape(-1, 1), pos[c_rows],
                         (c_rows + g0).to(torch.float64).reshape(-1, 1)], 1)
        got = comm.all_gather_rows(msg, comm.all_gather_ints([int(mine.numel())])[:, 0])
        order = got[:, 0].to(torch.int64)
        cpos = torch.empty((m, 3), dtype=torch.float64, device=dev)
        cpos[order] = got[:, 1:4]
        _tick("cd: centers")
        # class bounding box (sizes the hash grid like the single-device build)
        p_c = pos.contiguous() if len(classes) == 1 else pos[rows].contiguous()
        lo = p_c.min(0).values if my_n else torch.full((3,), float("inf"), dtype=torch.float64,
                                                         device=dev)
        hi = p_c.max(0).values if my_n else torch.full((3,), -float("inf"), dtype=torch.float64,
                                                         device=dev)
        bb = torch.cat([-lo, hi])
        comm.all_reduce_max_(bb)
        bounds = torch.cat([-bb[:3], bb[3:]]).cpu().numpy()
        assign = torch.empty(my_n, dtype=torch.int32, device=dev)
        if my_n:
            N.check(lib.vpg_assign_nearest(p_c.data_ptr(), my_n, cpos.contiguous().data_ptr(), m,
                                           bounds.ctypes.data, assign.data_ptr(), None, stream))
        _tick("cd: bbox+assign")
        a64 = assign.to(torch.int64)
        hist = torch.bincount(a64, minlength=m) if my_n else torch.zeros(m, dtype=torch.int64,
                                                                            device=dev)
        # group sizes and this shard's offset in every group: an exclusive
        # scan across the shards (no (world, m) all-gather)
        before, gsize = comm.exclusive_scan(hist)
        # rank of each row among its group's members (ascending global row)
        sv, srt = torch.sort(assign, stable=True)  # 32-bit keys: a 4-pass radix sort
        first = torch.cumsum(hist, 0) - hist
        lrank = torch.empty(my_n, dtype=torch.int64, device=dev)
        lrank[srt] = torch.arange(my_n, device=dev) - first[sv.to(torch.int64)]
        over = torch.nonzero(gsize > max_size).reshape(-1)
        n_over = int(over.numel())
        # reference numbering: non-empty groups in center order, then the
        # split-off groups of this class (clustering.py:87-93)
        nonempty = gsize > 0
        cid_of_j = torch.cumsum(nonempty.to(torch.int64), 0) - 1 + base
        n_ne = int(nonempty.sum())
        cl_sizes = gsize[nonempty].clone()
        cl_pos = cpos[nonempty].clone()
        is_over = torch.zeros(m, dtype=torch.bool, device=dev)
        is_over[over] = True
        # rows of the groups that need no split: cluster and rank at once
        # (dense where/index_copy, no boolean indexing and its host syncs;
        # the oversize groups' rows stay -1 until the split loop below)
        plain = ~is_over[a64]
        minus = torch.full_like(lrank, -1)
        row_cluster.index_copy_(0, rows, torch.where(plain, cid_of_j[a64], minus))
        row_rank.index_copy_(0, rows, torch.where(plain, before[a64] + lrank, minus))
        _tick("cd: groups")
        appended = []
        if n_over:
            om = torch.nonzero(is_over[a64]).reshape(-1)
            grow = (rows[om] + g0)
            mem = torch.cat([a64[om].to(torch.float64).reshape(-1, 1),
                             grow.to(torch.float64).reshape(-1, 1), p_c[om],
                             _sq_dist(p_c[om], cpos[a64[om]]).reshape(-1, 1)], 1)
            allm = comm.all_gather_rows(mem, comm.all_gather_ints([int(om.numel())])[:, 0])
            gj = allm[:, 0].to(torch.int64)
            gr = allm[:, 1].to(torch.int64)
            srt2 = group_member_order(gj, gr)
            allm, gj, gr = allm[srt2], gj[srt2], gr[srt2]
            crec = torch.empty(m, dtype=torch.int64, device=dev)
            crec[order] = got[:, 4].to(torch.int64)
            osz = gsize[over]
            ostart = torch.cumsum(osz, 0) - osz
            # slot of each group's center among its members (-1: not a member)
            cslot = torch.full((n_over,), -1, dtype=torch.int64, device=dev)
            hit = torch.nonzero(gr == crec[gj]).reshape(-1)
            if hit.numel():
                kk = torch.searchsorted(over, gj[hit])
                cslot[kk] = hit  # members ascending: one hit per group
            staged = int(allm.shape[0])
            ids_d = torch.arange(staged, dtype=torch.int32, device=dev)
            xyzd = allm[:, 2:6].t().contiguous()  # SoA rows, on the device
            _tick("cd: gather oversize")
            st = N.Pcg64State.from_generator(rng)
            cap = staged + n_over + 1
            o_n = ctypes.c_int64()
            o_b = np.zeros(cap, np.int64)
            o_s = np.zeros(cap, np.int64)
            o_c = np.zeros(cap, np.int64)
            nspl = ctypes.c_int64()
            sz_h = osz.cpu().numpy().astype(np.int64)
            cen_h = crec[over].cpu().numpy().astype(np.int64)
            cs_h = cslot.cpu().numpy().astype(np.int64)
            # first splits' bit rows on the device, the loop on the host
            N.check(lib.vpg_split_groups_device(
                ctypes.byref(st), ids_d.data_ptr(), xyzd[0].data_ptr(), xyzd[1].data_ptr(),
                xyzd[2].data_ptr(), xyzd[3].data_ptr(), n_over, sz_h.ctypes.data,
                cen_h.ctypes.data, cs_h.ctypes.data, max_size, cap, ctypes.byref(o_n),
                o_b.ctypes.data, o_s.ctypes.data, o_c.ctypes.data, ctypes.byref(nspl), stream))
            st.store_into(rng)
            _tick("cd: split loop")
            n_splits += nspl.value
            ng = o_n.value
            # final groups: members (staged index) in order; cluster ids: the
            # originals keep their slot among the non-empty groups, split-off
            # groups are appended
            # the final groups' ranges tile the staged array: each position's
            # group is the last range starting at or before it
            ids_t = ids_d.to(torch.int64)
            b_t = torch.as_tensor(o_b[:ng], device=dev)
            order_b = torch.argsort(b_t)
            posn = torch.arange(ids_t.numel(), device=dev)
            fg = order_b[torch.searchsorted(b_t[order_b], posn, right=True) - 1]
            fpos = posn - b_t[fg]
            member_idx = ids_t
            g_cid = torch.empty(ng, dtype=torch.int64, device=dev)
            g_cid[:n_over] = cid_of_j[over]
            g_cid[n_over:] = base + n_ne + torch.arange(ng - n_over, device=dev)
            # sizes / centers of the originals (shrunk) and the appended groups
            cl_sizes[(cid_of_j[over] - base)] = torch.as_tensor(o_s[:n_over], device=dev)
            center_rec = torch.as_tensor(o_c[:ng], device=dev)
            # (the originals keep their centers; a split-off group's center is
            # one of the class's oversize members)
            srt_gr, srt_i = torch.sort(gr)
            cidx = srt_i[torch.searchsorted(srt_gr, center_rec[n_over:])]
            appended = [(torch.as_tensor(o_s[n_over:ng], device=dev), allm[cidx, 2:5])]
            # my rows in oversize groups: their final group and rank
            mem_grow = gr[member_idx]
            my_lo, my_hi = g0, g0 + n
            mine2 = torch.nonzero((mem_grow >= my_lo) & (mem_grow < my_hi)).reshape(-1)
            lr = mem_grow[mine2] - g0
            row_cluster[lr] = g_cid[fg[mine2]]
            row_rank[lr] = fpos[mine2]
        sizes_all.append(cl_sizes)
        cpos_all.append(cl_pos)
        for sz, cp in appended:
            sizes_all.append(sz)
            cpos_all.append(cp)
        base += n_ne + sum(int(sz.numel()) for sz, _ in appended)
    sizes = torch.cat(sizes_all) if sizes_all else torch.zeros(0, dtype=torch.int64, device=dev)
    center_pos = torch.cat(cpos_all) if cpos_all else torch.zeros((0, 3), dtype=torch.float64,
                                                                  device=dev)
    _tick("cd: mapping")
    return GlobalClusters(sizes, center_pos, row_cluster, row_rank, n_splits)


def group_member_order(gj, gr):
    """Permutation ordering staged oversize members by (group gj, global row
    gr), both ascending (the split loop's `ostart`/`over` layout).  Two stable
    sorts instead of one packed int64 key: a packed `gj << 40 | gr` overflows
    once a class has 2^23 centers (C5 scale)."""
    import torch

    by_row = torch.argsort(gr, stable=True)
    return by_row[torch.argsort(gj[by_row], stable=True)]


# ------------------------------------------------------------ record payload
def _payload_columns():
    cols = []
    for name, width, code in N.RECORD_FIELDS:
        cols.append((name, width, code))
    cols += [("parent_ipt", 3, "f8"), ("has_child", 1, "i8"), ("grow", 1, "i8"),
             ("par_shard", 1, "i8"), ("par_row", 1, "i8"), ("dest_row", 1, "i8")]
    return cols


def _torch_dtype(code):
    import torch

    return {"f8": torch.float64, "i8": torch.int64, "i4": torch.int32, "u1": torch.uint8}[code]


def pack_payload(cols: dict, n: int):
    """Record columns -> (n, B) uint8: every column's bytes side by side (exact
    transport of every dtype, 354 bytes per record)."""
    import torch

    parts = []
    for name, width, code in _payload_columns():
        t = cols[name].reshape(n, width).contiguous()
        # explicit row width: a shard may send no rows at all
        parts.append(t.view(torch.uint8).reshape(n, width * t.element_size()))
    return torch.cat(parts, 1) if parts else None


def unpack_payload(p):
    import torch

    out, c = {}, 0
    for name, width, code in _payload_columns():
        dt = _torch_dtype(code)
        nb = width * torch.empty((), dtype=dt).element_size()
        if p.shape[0] == 0:  # no rows (a view of 0 bytes cannot change dtype)
            t = torch.empty((0, width), dtype=dt, device=p.device)
        else:
            # a fresh copy: a single row counts as contiguous whatever its
            # stride and offset, and a dtype view needs both aligned
            t = p[:, c:c + nb].clone(memory_format=torch.contiguous_format)
            t = t.view(-1).view(dt).reshape(p.shape[0], width)
        c += nb
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
        # the exact clustering, distributed (cluster_distributed)
        rng = np.random.default_rng(np.random.SeedSequence([seed & 0xFFFFFFFF, 0xC1A5]))
        g0 = int(self.row_off[me])
        gcl = cluster_distributed(comm, recs["pos"][:n_rec], recs["kind"][:n_rec],
                                  recs["class_id"][:n_rec], g0, cluster_size, rng)
        sizes = gcl.sizes
        m = int(sizes.numel())
        self.n_clusters_total = m
        self.n_splits = gcl.n_splits
        _tick("build: clustering")
        plan = plan_owners(sizes, gcl.center_pos, world)
        self.plan = plan
        dest_shard = plan.owner[gcl.row_cluster]
        dest_row = plan.local_start[gcl.row_cluster] + gcl.row_rank

        # this shard's records, with what the owner needs beyond them: the
        # continuation parent (record r-1 of the same path) is on this shard,
        # so its destination travels with the child
        n = n_rec
        cols = {name: recs[name][:n] for name, _, _ in N.RECORD_FIELDS}
        pidx = cols["path_idx"]
        has_child = torch.zeros(n, dtype=torch.int64, device="cuda")
        if n > 1:
            has_child[:-1] = (pidx[1:] == pidx[:-1]).to(torch.int64)
        parent_ipt = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
        par_shard = torch.full((n,), -1, dtype=torch.int64, device="cuda")
        par_row = torch.full((n,), -1, dtype=torch.int64, device="cuda")
        if n > 1:
            parent_ipt[1:] = cols["i_pt"][:-1]
            par_shard[1:] = dest_shard[:-1]
            par_row[1:] = dest_row[:-1]
        first = cols["depth"] == 0
        parent_ipt[first] = 0.0
        par_shard[first] = -1
        grow = torch.arange(g0, g0 + n, dtype=torch.int64, device="cuda")
        cols.update(parent_ipt=parent_ipt, has_child=has_child, grow=grow, par_shard=par_shard,
                    par_row=par_row, dest_row=dest_row)
        _tick("build: plan+cols")
        n_own = int(plan.rows[me])
        # rows that stay on this shard are placed field by field; only the
        # others travel, byte-packed, in one all-to-all
        own = {}
        for name, width, code in _payload_columns():
            shape = (n_own, width) if width > 1 else (n_own,)
            own[name] = torch.empty(shape, dtype=_torch_dtype(code), device="cuda")
        keep = dest_shard == me
        li = torch.nonzero(keep).reshape(-1)
        lr = dest_row[li]
        whole = lr.numel() == n_own  # every owned row is local (one shard)
        if whole:
            # placed in destination order: the destination rows are a
            # permutation, so its inverse (one scatter of indices) turns the
            # move into gathers of the sources (random reads, sequential writes)
            src = torch.empty(n_own, dtype=torch.int64, device="cuda")
            src[lr] = li
            for name, _, _ in _payload_columns():
                torch.index_select(cols[name], 0, src, out=own[name])
        else:
            for name, _, _ in _payload_columns():
                own[name][lr] = cols[name][li]
        if not comm.local:
            ri = torch.nonzero(~keep).reshape(-1)
            ds = dest_shard[ri]
            order = torch.argsort(ds, stable=True)
            send_counts = torch.bincount(ds, minlength=world).tolist() if ri.numel() else [0] * world
            sc = torch.tensor(send_counts, dtype=torch.int64, device="cuda").reshape(-1, 1)
            recv_counts = comm.all_to_all(sc, [1] * world, [1] * world).reshape(-1).tolist()
            sel = ri[order]
            payload = pack_payload({k: v[sel] for k, v in cols.items()}, int(sel.numel()))
            got = comm.all_to_all(payload, send_counts, recv_counts)
            if got is not None and got.shape[0]:
                recv = unpack_payload(got)
                rows_at = recv["dest_row"]
                for name, _, _ in _payload_columns():
                    own[name][rows_at] = recv[name]
        _tick("build: records to owners")
        self.own = own
        self.n = n_own

        # continuation parents: local row, or a halo slot for a remote one
        parent = torch.full((n_own,), -1, dtype=torch.int64, device="cuda")
        rows_with = torch.nonzero(own["par_shard"] >= 0).reshape(-1)
        p_shard = own["par_shard"][rows_with]
        p_row = own["par_row"][rows_with]
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

        _tick("build: unpack+halo")
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
        _tick("build: build_local")
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
        # the residual maxima are IEEE bit patterns of non-negative floats
        # (NaN above +inf): an integer max reduces them across the shards
        red_i = _view(v.red, ((iterations + 1) * 8,), "<i4")
        for t in range(iterations):
            N.check(lib.vpg_solve_step(self.handle, t, stream))
            if not self.comm.local:
                i_out = _view(v.ibuf[(t + 1) & 1], (rows, 4), "<f4")
                self.halo.exchange(i_out)
                self.comm.all_reduce_max_(red_i[t * 8:t * 8 + _RESIDUAL_WORDS])
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
    pt_image: np.ndarray = None  # the frame's PT image (render_pg's pt_image)


def render_pg_sharded(scene, config: RenderConfig, comm: ShardComm | None = None,
                      keep_graph: bool = True) -> ShardedRender:
    """render_pg (pipeline.py:25-42) over the shards of `comm` (default: the
    initialised torch.distributed group, or a single shard)."""
    from paper_2404_11894_b200.transport.tracer import trace_records_device

    comm = comm or ShardComm()
    packed = pack_scene(scene)
    w, h, spp = packed.width, packed.height, int(config.spp)
    ranges = pixel_ranges(w * h, comm.world)
    p0, p1 = ranges[comm.rank]
    recs, paths, n_rec = trace_records_device(scene, config, ((p0 * spp), (p1 - p0) * spp))
    rst, pst = _structs(recs, paths, n_rec, (p1 - p0) * spp)
    if config.extra_direct_samples > 0:
        # record_extra_direct (pipeline.py:28-29) on this shard's paths, keyed
        # by the frame's path index
        N.check(N.lib().vpg_extra_direct_range(
            ctypes.byref(packed.device()), ctypes.byref(rst), ctypes.byref(pst), p0 * spp,
            int(np.int64(config.seed)), int(config.extra_direct_samples), N.stream_handle()))
    else:
        paths["extra_direct"].copy_(paths["direct0"])
    if config.dump_records:
        _dump_frame(comm, config.dump_records, recs, paths, n_rec, w, h, spp)
    g = ShardedPathGraph.build(comm, recs, n_rec, config.cluster_size, seed=config.seed)
    g.pix_ranges = ranges
    sol = g.solve(config.iterations, config.tol)
    if config.residual_csv and comm.rank == 0:
        from paper_2404_11894_b200.pathgraph.solve import write_residual_csv

        write_residual_csv(config.residual_csv, sol.residuals)
    if config.aggregate_direct:
        mode = N.DIRECT_AGGREGATED
    else:
        mode = N.DIRECT_EXTRA if config.extra_direct_samples > 0 else N.DIRECT_PT
    img = g.splat(paths, recs, (p0, p1), w, h, spp, mode)
    # splat_pt_image (records.py:259-265) of this shard's pixels, gathered
    import torch

    pt = torch.zeros(((p1 - p0) + 1, 3), dtype=torch.float64, device="cuda")
    if p1 > p0:
        N.check(N.lib().vpg_splat_pt(ctypes.byref(pst), p1 - p0, 1, spp, pt.data_ptr(),
                                     N.stream_handle()))
    pt_full = comm.all_gather_rows(pt[:p1 - p0], [b - a for a, b in ranges]).reshape(h, w, 3)
    total = int(g.row_off[-1])
    return ShardedRender(image=img.cpu().numpy(), residuals=sol.residuals,
                         iterations=sol.iterations, graph=g if keep_graph else None,
                         n_records=n_rec, n_records_total=total,
                         pt_image=pt_full.cpu().numpy())


def _structs(recs: dict, paths: dict, n_rec: int, n_paths: int):
    """vpg_records / vpg_paths views of a shard's device tensors."""
    rst, pst = N.Records(), N.Paths()
    rst.n, pst.n = n_rec, n_paths
    for name, _, _ in N.RECORD_FIELDS:
        t = recs[name]
        setattr(rst, name, t.data_ptr() if t.numel() else None)
    for name, _, _ in N.PATH_FIELDS:
        t = paths[name]
        setattr(pst, name, t.data_ptr() if t.numel() else None)
    return rst, pst


def _dump_frame(comm, path, recs, paths, n_rec, w, h, spp):
    """save_records (records.py:191-217) of the whole frame: the shards'
    records in shard order are the frame's (contiguous path ranges), path
    rows re-based to frame record offsets; rank 0 writes the file."""
    import torch

    from paper_2404_11894_b200.transport.records import PathSoA, RecordSoA, TraceOutput, save_records

    counts = comm.all_gather_ints([n_rec])[:, 0]
    base = int(counts[: comm.rank].sum())
    n_paths = int(paths["rec_start"].shape[0])
    pcounts = comm.all_gather_ints([n_paths])[:, 0]
    rec_all, path_all = {}, {}
    for name, _, _ in N.RECORD_FIELDS:
        rec_all[name] = comm.all_gather_rows(recs[name][:n_rec], counts)
    for name, _, _ in N.PATH_FIELDS:
        t = paths[name]
        if name == "rec_start":
            t = t + base
        path_all[name] = comm.all_gather_rows(t, pcounts)
    if comm.rank == 0:
        out = TraceOutput(None, RecordSoA(**{k: v.cpu().numpy() for k, v in rec_all.items()}),
                          PathSoA(**{k: v.cpu().numpy() for k, v in path_all.items()}), w, h, spp)
        save_records(path, out)

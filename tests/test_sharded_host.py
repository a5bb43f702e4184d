"""Host logic of the sharded (multi-GPU) path on CPU: ownership plan, record
destinations, and the per-iteration halo exchange, with world_size-2 gloo
process groups.  The per-shard fixed-point step is emulated in float64 torch
on the CPU (the device kernel is covered by tests/test_gpu_sharded.py); the
sharded run must equal the single-process run bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2404_11894_b200.pathgraph import sharded as S


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(seed=0, n_paths=300, k=8):
    """Random paths and clusters (cluster members ascending, like the build)."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 7, n_paths)
    path_idx = np.repeat(np.arange(n_paths), lens)
    n = path_idx.size
    depth = np.concatenate([np.arange(c) for c in lens])
    m = (n + k - 1) // k
    cid = rng.integers(0, m, n)
    cid[:m] = np.arange(m)  # no empty cluster
    order = np.argsort(cid, kind="stable")
    sizes = np.bincount(cid, minlength=m)
    cl_off = np.concatenate([[0], np.cumsum(sizes)])
    centers = order[cl_off[:-1]]
    pos = rng.random((n, 3))
    # per-row data of the emulated iteration
    a = rng.random(n) * 0.5
    b = rng.random(n)
    i0 = rng.random(n)
    w = {k_: rng.random((sizes[k_], sizes[k_])) / max(sizes[k_], 1) for k_ in range(m)}
    return dict(path_idx=path_idx, depth=depth, perm=order, cl_off=cl_off, sizes=sizes,
                centers=centers, pos=pos, a=a, b=b, i0=i0, w=w, n=n, m=m)


def _destinations(P, plan):
    """(shard, row) of every record: its cluster's shard, the cluster's first
    row there plus the record's rank among the members (as the sharded build
    derives them from cluster_distributed's row_cluster/row_rank)."""
    n, m = P["n"], P["m"]
    k_of = np.empty(n, np.int64)
    rank = np.empty(n, np.int64)
    for k in range(m):
        mem = P["perm"][P["cl_off"][k]:P["cl_off"][k + 1]]
        k_of[mem] = k
        rank[mem] = np.arange(mem.size)
    k_of, rank = torch.tensor(k_of), torch.tensor(rank)
    return plan.owner[k_of], plan.local_start[k_of] + rank


def _global_iterate(P, T):
    """Reference emulation: I[parent(r)] = a[r] * (W I)[r] + b[r], record order."""
    n = P["n"]
    has_par = P["depth"] > 0
    I = torch.tensor(P["i0"])
    a, b = torch.tensor(P["a"]), torch.tensor(P["b"])
    for _ in range(T):
        new = I.clone()
        for k in range(P["m"]):
            mem = P["perm"][P["cl_off"][k]:P["cl_off"][k + 1]]
            acc = torch.tensor(P["w"][k]) @ I[torch.tensor(mem)]  # same op as the shards'
            for r, ac in zip(mem, acc):
                if has_par[r]:
                    new[r - 1] = a[r] * ac + b[r]
        I = new
    return I.numpy()


def _worker(rank, world, port, T, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = S.ShardComm()
        P = _problem()
        n, m = P["n"], P["m"]
        # path-aligned row ranges, like the pixel ranges of the tracer
        cuts = [0] + [int(np.searchsorted(P["path_idx"], P["path_idx"][-1] * r // world))
                      for r in range(1, world)] + [n]
        counts = [cuts[r + 1] - cuts[r] for r in range(world)]
        sizes = torch.tensor(P["sizes"])
        plan = S.plan_owners(sizes, torch.tensor(P["pos"][P["centers"]]), world)
        dest_shard, dest_row = _destinations(P, plan)
        # every shard owns a permutation of its rows; members stay ascending
        mine = torch.nonzero(dest_shard == rank).reshape(-1)
        assert sorted(dest_row[mine].tolist()) == list(range(plan.rows[rank]))
        for k in range(m):
            mem = P["perm"][P["cl_off"][k]:P["cl_off"][k + 1]]
            rows = dest_row[torch.tensor(mem)]
            assert torch.all(rows[1:] - rows[:-1] == 1)
            assert len(set(dest_shard[torch.tensor(mem)].tolist())) == 1
        # move this shard's rows to their owners (payload: global row)
        g0 = cuts[rank]
        grow = torch.arange(g0, cuts[rank + 1])
        dst = dest_shard[grow]
        order = torch.argsort(dst, stable=True)
        send_counts = torch.bincount(dst, minlength=world).tolist()
        sc = torch.tensor(send_counts, dtype=torch.int64).reshape(-1, 1)
        recv_counts = comm.all_to_all(sc, [1] * world, [1] * world).reshape(-1).tolist()
        got = comm.all_to_all(torch.stack([grow, dest_row[grow]], 1)[order], send_counts,
                              recv_counts)
        own = torch.empty(plan.rows[rank], dtype=torch.int64)
        own[got[:, 1]] = got[:, 0]
        # halo plan exactly as ShardedPathGraph.build
        depth = torch.tensor(P["depth"])[own]
        rows_with = torch.nonzero(depth > 0).reshape(-1)
        par_g = own[rows_with] - 1
        p_shard, p_row = dest_shard[par_g], dest_row[par_g]
        local = p_shard == rank
        parent = torch.full((own.numel(),), -1, dtype=torch.int64)
        parent[rows_with[local]] = p_row[local]
        halo = S.HaloExchange(comm, own.numel(), p_shard[~local], p_row[~local],
                              rows_with[~local])
        parent[halo.child_rows] = own.numel() + torch.arange(halo.n_halo)
        # emulated iterations on this shard's clusters
        a = torch.tensor(P["a"])[own]
        b = torch.tensor(P["b"])[own]
        I = torch.zeros(own.numel() + halo.n_halo, dtype=torch.float64)
        I[:own.numel()] = torch.tensor(P["i0"])[own]
        own_k = plan.order[plan.owner[plan.order] == rank].tolist()
        for _ in range(T):
            new = I.clone()
            q = 0
            for k in own_k:
                s = int(P["sizes"][k])
                acc = torch.tensor(P["w"][k]) @ I[q:q + s]
                for j in range(s):
                    if parent[q + j] >= 0:
                        new[parent[q + j]] = a[q + j] * acc[j] + b[q + j]
                q += s
            halo.exchange(new.reshape(-1, 1))
            I = new
        res = torch.zeros(n, dtype=torch.float64)
        full_rows = comm.all_gather_rows(own, comm.all_gather_ints([own.numel()])[:, 0])
        full_vals = comm.all_gather_rows(I[:own.numel()], comm.all_gather_ints([own.numel()])[:, 0])
        res[full_rows] = full_vals
        if rank == 0:
            out_q.put((res.numpy(), halo.n_halo + sum(halo.recv_counts)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_exchange_matches_single_process(world):
    T = 4
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.spawn(_worker, args=(world, _free_port(), T, q), nprocs=world, join=True)
    res, crossing = q.get()
    ref = _global_iterate(_problem(), T)
    assert crossing > 0, "the test problem must have cross-shard edges"
    np.testing.assert_array_equal(res, ref)


def test_plan_owners_balances_cost_and_is_contiguous():
    P = _problem(seed=3, n_paths=2000)
    sizes = torch.tensor(P["sizes"])
    for world in (1, 2, 4, 8):
        plan = S.plan_owners(sizes, torch.tensor(P["pos"][P["centers"]]), world)
        own_o = plan.owner[plan.order]
        assert torch.all(own_o[1:] >= own_o[:-1]), "shards are contiguous in Morton order"
        assert sum(plan.rows) == P["n"]
        cost = (sizes * sizes + 16 * sizes).double()
        per = torch.zeros(world, dtype=torch.float64).index_add_(0, plan.owner, cost)
        assert float(per.max() / per.mean()) < 1.1


def test_pixel_ranges_cover_every_pixel_once():
    for n_pix, world in [(10, 3), (4096, 8), (1, 2)]:
        r = S.pixel_ranges(n_pix, world)
        assert r[0][0] == 0 and r[-1][1] == n_pix
        assert all(r[i][1] == r[i + 1][0] for i in range(world - 1))


def test_morton_order_is_z_order():
    q = torch.tensor([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 1], [2, 0, 0]])
    assert S.morton3(q).tolist() == [0, 1, 2, 4, 7, 8]


def test_group_member_order_beyond_2_pow_23_centers():
    """Oversize members sort by (group, global row) even when a class has more
    than 2^23 centers and rows beyond 2^40 (a packed gj<<40|gr key wraps)."""
    import torch

    from paper_2404_11894_b200.pathgraph.sharded import group_member_order

    rng = np.random.default_rng(7)
    n = 20000
    gj = torch.as_tensor(rng.integers(0, 1 << 25, n) | np.where(rng.random(n) < 0.5, 1 << 24, 0))
    gr = torch.as_tensor(rng.integers(0, 1 << 41, n))
    gj[:50] = (1 << 25) - 1  # the top groups: a packed key would make them negative
    o = group_member_order(gj, gr)
    expect = np.lexsort((gr.numpy(), gj.numpy()))
    assert np.array_equal(o.numpy(), expect)


def _scan_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = S.ShardComm()
        bad = []
        for m in (1, 5, 1000, 1003):
            v = torch.as_tensor(np.random.default_rng(rank * 100 + m).integers(0, 50, m))
            before, total = comm.exclusive_scan(v)
            parts = [torch.empty_like(v) for _ in range(world)]
            dist.all_gather(parts, v)
            want_b = sum(parts[:rank], torch.zeros_like(v))
            want_t = sum(parts, torch.zeros_like(v))
            if not (torch.equal(before, want_b) and torch.equal(total, want_t)):
                bad.append(m)
        out_q.put((rank, bad))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_exclusive_scan_of_group_sizes(world):
    """The group-size exchange of the distributed clustering (all-to-all scan
    instead of an all-gather): every shard gets the sum over the shards
    before it and the total."""
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.spawn(_scan_worker, args=(world, _free_port(), q), nprocs=world, join=True)
    res = [q.get() for _ in range(world)]
    assert all(not bad for _, bad in res), res


@pytest.mark.parametrize("n", [0, 1, 7])
def test_record_payload_round_trip(n):
    """The byte payload the owner all-to-all moves: every column's bytes back
    exactly, including a shard that sends no rows."""
    import torch

    from paper_2404_11894_b200.pathgraph.sharded import (_payload_columns, _torch_dtype,
                                                          pack_payload, unpack_payload)

    g = torch.Generator().manual_seed(n)
    cols = {}
    for name, width, code in _payload_columns():
        dt = _torch_dtype(code)
        shape = (n, width) if width > 1 else (n,)
        if dt.is_floating_point:
            cols[name] = torch.randn(shape, generator=g, dtype=dt)
        else:
            cols[name] = torch.randint(0, 100, shape, generator=g).to(dt)
    back = unpack_payload(pack_payload(cols, n))
    for name, width, _ in _payload_columns():
        assert torch.equal(back[name].reshape(cols[name].shape), cols[name]), name

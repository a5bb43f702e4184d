"""The sharded (multi-GPU row-partition) path on the device: 1, 2 and 3 shards
must give bit-identical images and solutions to the single-GPU render_pg.

With one GPU on the test box the shards are processes sharing cuda:0 over a
gloo group: every exchange is host-staged between kernel launches, so no
kernel waits on another process (B200_PROFILING.md's rule for emulating
ranks on fewer GPUs).  NCCL on one GPU per shard runs the same code."""

import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = {
    "c1floor": dict(res=(24, 24), spp=2, max_depth=16, K=32, iters=6, seed=1),
    "cloud": dict(res=(20, 20), spp=4, max_depth=64, K=16, iters=5, seed=2),
    # small K: many oversize groups and deep split chains in both classes
    "c1floor_k4": dict(res=(16, 16), spp=2, max_depth=16, K=4, iters=4, seed=5),
}


def _scene(name, res):
    from paper_2404_11894_b200 import scenes as S

    if name.startswith("c1floor"):
        return S.scene_c1(res, floor=True)
    return S.scene_c2(res, grid_n=16)


def _config(c):
    from paper_2404_11894_b200.harness.config import RenderConfig

    return RenderConfig(mode="pg", spp=c["spp"], max_depth=c["max_depth"], seed=c["seed"],
                        cluster_size=c["K"], iterations=c["iters"], tol=0.0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard_worker(rank, world, port, name, out_path):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2404_11894_b200.pathgraph.sharded import ShardComm, render_pg_sharded

        c = CASES[name]
        out = render_pg_sharded(_scene(name, c["res"]), _config(c), ShardComm())
        inc, ibar = out.graph.gather_solution()
        if rank == 0:
            np.savez(out_path, image=out.image, incoming=inc.cpu().numpy(),
                     i_bar=ibar.cpu().numpy(), residuals=np.array(out.residuals),
                     halo=out.graph.halo.n_halo, n_total=out.n_records_total,
                     n_clusters=out.graph.n_clusters_total, n_splits=out.graph.n_splits)
    finally:
        dist.destroy_process_group()


def _single(name):
    from paper_2404_11894_b200.pathgraph import render_pg

    c = CASES[name]
    pg = render_pg(_scene(name, c["res"]), _config(c))
    return pg


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_render_is_bit_identical(cuda, name, world):
    import torch.multiprocessing as mp

    ref = _single(name)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "shard0.npz")
        if world == 1:
            from paper_2404_11894_b200.pathgraph.sharded import ShardComm, render_pg_sharded

            c = CASES[name]
            out = render_pg_sharded(_scene(name, c["res"]), _config(c), ShardComm())
            inc, ibar = out.graph.gather_solution()
            got = dict(image=out.image, incoming=inc.cpu().numpy(), i_bar=ibar.cpu().numpy(),
                       residuals=np.array(out.residuals), halo=0, n_total=out.n_records_total,
                       n_clusters=out.graph.n_clusters_total, n_splits=out.graph.n_splits)
        else:
            mp.spawn(_shard_worker, args=(world, _free_port(), name, path), nprocs=world,
                     join=True)
            got = dict(np.load(path))
    assert int(got["n_total"]) == ref.trace.records.n
    info = ref.graph.info()
    assert int(got["n_clusters"]) == info["n_clusters"]
    assert int(got["n_splits"]) == info["n_splits"]
    if world > 1:
        assert int(got["halo"]) > 0, "expected continuation edges across shards"
    np.testing.assert_array_equal(got["image"], ref.image)
    np.testing.assert_array_equal(got["incoming"], ref.result.incoming)
    np.testing.assert_array_equal(got["i_bar"], ref.result.i_bar)
    np.testing.assert_array_equal(got["residuals"], np.array(ref.result.residuals))


def _feature_config(tmp, tag):
    from paper_2404_11894_b200.harness.config import RenderConfig

    return RenderConfig(mode="pg", spp=2, max_depth=16, seed=3, cluster_size=16, iterations=5,
                        tol=0.0, extra_direct_samples=3,
                        residual_csv=os.path.join(tmp, f"res_{tag}.csv"),
                        dump_records=os.path.join(tmp, f"dump_{tag}.vpgr"))


def _feature_worker(rank, world, port, tmp):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2404_11894_b200 import scenes as S
        from paper_2404_11894_b200.pathgraph.sharded import ShardComm, render_pg_sharded

        out = render_pg_sharded(S.scene_mixed((14, 14)), _feature_config(tmp, "sharded"),
                                ShardComm(), keep_graph=False)
        if rank == 0:
            np.savez(os.path.join(tmp, "sharded.npz"), image=out.image, pt=out.pt_image)
    finally:
        dist.destroy_process_group()


def test_sharded_render_pg_config_features(cuda):
    """render_pg's config flags on the sharded path (pipeline.py:28-36):
    extra_direct_samples (streams keyed by the frame's path index),
    dump_records (the whole frame, rank 0), residual_csv, and the PT image --
    all equal to the single-GPU render_pg, over 2 shards."""
    import torch.multiprocessing as mp

    from paper_2404_11894_b200 import scenes as S
    from paper_2404_11894_b200.pathgraph import render_pg

    with tempfile.TemporaryDirectory() as d:
        ref = render_pg(S.scene_mixed((14, 14)), _feature_config(d, "single"))
        mp.spawn(_feature_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        got = np.load(os.path.join(d, "sharded.npz"))
        np.testing.assert_array_equal(got["image"], ref.image)
        np.testing.assert_array_equal(got["pt"], ref.pt_image)
        assert open(os.path.join(d, "res_sharded.csv")).read() == \
            open(os.path.join(d, "res_single.csv")).read()
        assert open(os.path.join(d, "dump_sharded.vpgr"), "rb").read() == \
            open(os.path.join(d, "dump_single.vpgr"), "rb").read()


def _loopback_worker(rank, world, port, name, out_path):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", 0))
    try:
        from paper_2404_11894_b200.pathgraph.sharded import ShardComm, render_pg_sharded

        comm = ShardComm(loopback=True)
        assert comm.backend == "nccl" and not comm.staged and not comm.local
        c = CASES[name]
        out = render_pg_sharded(_scene(name, c["res"]), _config(c), comm)
        inc, ibar = out.graph.gather_solution()
        np.savez(out_path, image=out.image, incoming=inc.cpu().numpy(), i_bar=ibar.cpu().numpy(),
                 residuals=np.array(out.residuals))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["cloud", "c1floor_k4"])
def test_nccl_collectives_single_rank_loopback(cuda, name):
    """Every collective of the N > 1 path through NCCL itself (a one-rank
    NCCL group with the collectives looped back instead of skipped): device
    tensors in all_to_all_single / all_gather / all_reduce(MAX) of the
    residual bit patterns, the exclusive scan, the halo exchange -- the
    result stays bit-identical to render_pg.  (Two NCCL ranks cannot share
    the one GPU of the test pool.)"""
    import torch.multiprocessing as mp

    ref = _single(name)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "loopback.npz")
        mp.spawn(_loopback_worker, args=(1, _free_port(), name, path), nprocs=1, join=True)
        got = dict(np.load(path))
    np.testing.assert_array_equal(got["image"], ref.image)
    np.testing.assert_array_equal(got["incoming"], ref.result.incoming)
    np.testing.assert_array_equal(got["i_bar"], ref.result.i_bar)
    np.testing.assert_array_equal(got["residuals"], np.array(ref.result.residuals))

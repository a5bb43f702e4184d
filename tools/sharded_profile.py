"""Where a single-shard ShardedPathGraph.build spends its (host) time."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import torch
from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.pathgraph.sharded import ShardComm, ShardedPathGraph
from paper_2404_11894_b200.scenes import WORKLOADS
from paper_2404_11894_b200.transport.tracer import trace_records_device

wl = WORKLOADS["C2"]
cfg = RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0)
scene = wl.scene()
recs, paths, n = trace_records_device(scene, cfg)
comm = ShardComm()
for _ in range(2):
    g = ShardedPathGraph.build(comm, recs, n, 32); del g
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
g = ShardedPathGraph.build(comm, recs, n, 32)
torch.cuda.synchronize()
pr.disable()
print("build ms", (time.perf_counter() - t0) * 1e3)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)

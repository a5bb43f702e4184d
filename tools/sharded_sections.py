import sys, time
sys.path.insert(0, ".")
import torch
from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.pathgraph import sharded as SH
from paper_2404_11894_b200.scenes import WORKLOADS
from paper_2404_11894_b200.transport.tracer import trace_records_device
wl = WORKLOADS["C2"]
cfg = RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0)
recs, paths, n = trace_records_device(wl.scene(), cfg)
comm = SH.ShardComm()
# time sections of cluster_distributed by monkeypatching the native calls
import paper_2404_11894_b200._native as N
lib = N.lib()
times = {}
def wrap(name):
    f = getattr(lib, name)
    def g(*a):
        torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(*a); torch.cuda.synchronize()
        times[name] = times.get(name, 0) + (time.perf_counter() - t0) * 1e3
        return r
    return g
class L:
    def __getattr__(self, k):
        if k.startswith("vpg_rng_choice") or k in ("vpg_assign_nearest", "vpg_split_groups_soa", "vpg_graph_build_local"):
            return wrap(k)
        return getattr(lib, k)
N.lib = lambda: L()
for _ in range(3):
    times.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g = SH.ShardedPathGraph.build(comm, recs, n, 32)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print("build ms", round((t1 - t0) * 1e3, 2), {k: round(v, 2) for k, v in times.items()})
    del g

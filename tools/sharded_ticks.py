"""Section times of one sharded build + solve at world 1 (VPG_SHARD_TIMING=1)."""
import os
import sys
sys.path.insert(0, ".")
os.environ["VPG_SHARD_TIMING"] = "1"
import torch
from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.pathgraph import sharded as SH
from paper_2404_11894_b200.scenes import WORKLOADS
from paper_2404_11894_b200.transport.tracer import trace_records_device

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
cfg = RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0)
recs, paths, n = trace_records_device(wl.scene(), cfg)
comm = SH.ShardComm()
for rep in range(3):
    torch.cuda.synchronize()
    print(f"--- rep {rep}", flush=True)
    g = SH.ShardedPathGraph.build(comm, recs, n, 32, seed=0)
    g.solve(wl.iterations, 0.0)
    torch.cuda.synchronize()
    del g

import sys, time
sys.path.insert(0, ".")
import torch
from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.scenes import WORKLOADS
from paper_2404_11894_b200.transport import render_pt
wl = WORKLOADS["C2"]
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = render_pt(wl.scene(), RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0), with_records=False)
    torch.cuda.synchronize(); print("image-only C2", round(1e3 * (time.perf_counter() - t0), 2), "ms")

"""Where a record-capturing render_pt spends its time (device kernels vs host)."""
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_2404_11894_b200 import _native as N
from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.scenes import WORKLOADS
from paper_2404_11894_b200.transport import render_pt

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
cfg = RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0)
scene = wl.scene()
for rep in range(3):
    torch.cuda.synchronize()
    N.profile_reset(); N.profile(rep == 2)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    out = render_pt(scene, cfg, with_records=True)
    e1.record(); torch.cuda.synchronize()
    print(f"rep {rep}: events {e0.elapsed_time(e1):.2f} ms, wall {1e3*(time.perf_counter()-t0):.2f} ms, n={out.records.n}")
prof = N.profile_read(); N.profile(False)
for k, (c, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:30s} {c:3d} {ms:9.3f} ms")

"""Device times of the tracing kernels of one frame in each mode: record-free
image, single-pass capture, two-pass count + fill (diagnostic)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2404_11894_b200 import _native as N
from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.scenes import WORKLOADS
from paper_2404_11894_b200.transport import render_pt
from paper_2404_11894_b200.transport.tracer import trace_records_device
for name in sys.argv[1:]:
    wl = WORKLOADS[name]
    cfg = RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0)
    scene = wl.scene()
    for rep in range(2):
        torch.cuda.synchronize(); N.profile_reset(); N.profile(rep == 1)
        render_pt(scene, cfg, with_records=False)
        render_pt(scene, cfg, with_records=True)
        trace_records_device(scene, cfg, capture=False)
        torch.cuda.synchronize()
    prof = N.profile_read(); N.profile(False)
    print(name, {k: round(v[1], 2) for k, v in prof.items() if 'trace' in k})

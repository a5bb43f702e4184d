import sys
sys.path.insert(0, ".")
import torch
from paper_2404_11894_b200 import _native as N
from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.scenes import WORKLOADS
from paper_2404_11894_b200.transport import render_pt
wl = WORKLOADS[sys.argv[1]]
cfg = RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0)
scene = wl.scene()
for rep in range(3):
    torch.cuda.synchronize(); N.profile_reset(); N.profile(rep == 2)
    img = render_pt(scene, cfg, with_records=False).image
    torch.cuda.synchronize()
prof = N.profile_read(); N.profile(False)
for k, (c, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:30s} {c:3d} {ms:9.3f} ms")

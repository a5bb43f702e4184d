"""Device time of record_extra_direct (tracer.py:105-127) on a workload's
record set: diagnostic for the k_extra_direct kernel."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2404_11894_b200 import _native as N  # noqa: E402
from paper_2404_11894_b200.harness.config import RenderConfig  # noqa: E402
from paper_2404_11894_b200.scenes import WORKLOADS  # noqa: E402
from paper_2404_11894_b200.transport import record_extra_direct, render_pt  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
n_extra = int(sys.argv[2]) if len(sys.argv) > 2 else 4
scene = wl.scene()
out = render_pt(scene, RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0), with_records=True)
for rep in range(3):
    torch.cuda.synchronize()
    N.profile_reset()
    N.profile(rep == 2)
    ed = record_extra_direct(scene, out, n_extra, seed=1)
    torch.cuda.synchronize()
prof = N.profile_read()
N.profile(False)
print({k: round(v[1], 3) for k, v in prof.items()}, float(abs(ed).sum()))

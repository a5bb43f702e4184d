"""sha256 and time of record-free PT images (render_pt(with_records=False)) for
bit-level A/B of the image kernels: run once per library variant."""
import hashlib
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_11894_b200.harness.config import RenderConfig  # noqa: E402
from paper_2404_11894_b200.scenes import WORKLOADS  # noqa: E402
from paper_2404_11894_b200.transport import render_pt  # noqa: E402

out = {}
for name in sys.argv[1:]:
    wl = WORKLOADS[name]
    cfg = RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0)
    scene = wl.scene()
    ms = []
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        img = render_pt(scene, cfg, with_records=False).image
        torch.cuda.synchronize()
        ms.append(1e3 * (time.perf_counter() - t0))
    out[name] = {"sha": hashlib.sha256(np.ascontiguousarray(img).tobytes()).hexdigest()[:16],
                 "ms": round(min(ms), 2)}
print(json.dumps(out))

"""sha256 of every record and path field of a captured render_pt (bit-level A/B
of tracer changes: run once per library variant, VPG_LIB_VARIANT=...)."""
import hashlib
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2404_11894_b200.harness.config import RenderConfig  # noqa: E402
from paper_2404_11894_b200.scenes import WORKLOADS  # noqa: E402
from paper_2404_11894_b200.transport import render_pt  # noqa: E402

out = {}
for name in sys.argv[1:]:
    wl = WORKLOADS[name]
    t = render_pt(wl.scene(), RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0),
                  with_records=True)
    h = {}
    for k, v in t.records.host_arrays().items():
        h["rec." + k] = hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()[:16]
    for k, v in t.paths.host_arrays().items():
        h["path." + k] = hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()[:16]
    h["image"] = hashlib.sha256(np.ascontiguousarray(t.image).tobytes()).hexdigest()[:16]
    out[name] = h
print(json.dumps(out))

"""Capacity and per-vertex rate on a record set larger than C4 on one GPU
(the C4 scene at a higher resolution): trace, build + 16 iterations timed with
CUDA events, peak device memory.  The per-GPU share of C5 at 8 GPUs is
~130 M vertices; this checks that such a share fits the 180 GB and keeps
C4's rate."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2404_11894_b200 import _native as N  # noqa: E402
from paper_2404_11894_b200 import scenes as S  # noqa: E402
from paper_2404_11894_b200.harness.config import RenderConfig  # noqa: E402
from paper_2404_11894_b200.pathgraph import build_graph, solve  # noqa: E402
from paper_2404_11894_b200.transport import render_pt  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 1448
cfg = RenderConfig(spp=16, max_depth=64, seed=0)
scene = S.scene_c4((side, side))
t0 = time.perf_counter()
out = render_pt(scene, cfg, with_records=True)
torch.cuda.synchronize()
trace_s = time.perf_counter() - t0
# the capture scratch (320 B per record) and torch's cached blocks back to
# the device before the native build allocates
from paper_2404_11894_b200.transport.tracer import release_scratch  # noqa: E402

release_scratch()
torch.cuda.empty_cache()
n = out.records.n
ms = []
for rep in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    g = build_graph(out, 32, seed=0)
    solve(g, iterations=16, tol=0.0)
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
    del g
free, total = torch.cuda.mem_get_info()
print(json.dumps({"resolution": side, "vertices": n, "trace_s": round(trace_s, 2),
                  "step_ms": [round(x, 2) for x in ms],
                  "vertices_per_s": n / (min(ms[1:]) * 1e-3),
                  "torch_peak_gb": round(torch.cuda.max_memory_allocated() / 1e9, 1),
                  "device_used_gb_after": round((total - free) / 1e9, 1)}))

"""Where the end-to-end (host records -> image) time goes."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.scenes import WORKLOADS
from paper_2404_11894_b200.transport import render_pt
from paper_2404_11894_b200.transport.records import PathSoA, RecordSoA, TraceOutput
from paper_2404_11894_b200.pathgraph.pipeline import solve_from_records

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
cfg = RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0)
tr = render_pt(wl.scene(), cfg, with_records=True)
W, H = tr.width, tr.height
hr = RecordSoA(**tr.records.host_arrays()).pin_memory()
hp = PathSoA(**tr.paths.host_arrays()).pin_memory()
del tr

def fresh():
    t = TraceOutput(None, RecordSoA(**hr.host_arrays()), PathSoA(**hp.host_arrays()), W, H, wl.spp)
    t.records._pinned = hr._pinned
    t.paths._pinned = hp._pinned
    return t

for rep in range(3):
    t = fresh()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    t.records.upload_async(); t.paths.upload_async()
    t.records.device(); t.paths.device()
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"upload only: {(t1-t0)*1e3:.1f} ms")
for rep in range(3):
    t = fresh()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    img, g, r = solve_from_records(t, 32, iterations=wl.iterations, tol=0.0)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"solve_from_records: {(t1-t0)*1e3:.1f} ms")
    del g, r, t

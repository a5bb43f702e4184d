"""VPGR dump I/O at bench size: trace C2 on the device, then time the device
save (pack on device + chunked D2H + write), the host load (numpy), and the
device load (chunked read + H2D + device unpack).  Prints one JSON line."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2404_11894_b200 import scenes as S  # noqa: E402
from paper_2404_11894_b200.harness.config import RenderConfig  # noqa: E402
from paper_2404_11894_b200.transport import load_records, render_pt, save_records  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t0


def main():
    wl = S.WORKLOADS["C2"]
    cfg = RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0)
    t = render_pt(wl.scene(), cfg, with_records=True)
    n = t.records.n
    d = tempfile.mkdtemp()
    p = os.path.join(d, "c2.vpgr")
    out = {"n_records": n}
    for k in range(2):
        _, out["save_device_s"] = timed(lambda: save_records(p, t))
    out["file_bytes"] = os.path.getsize(p)
    for k in range(2):
        _, out["load_host_s"] = timed(lambda: load_records(p))
    for k in range(2):
        back, out["load_device_s"] = timed(lambda: load_records(p, device=True))
    for k in range(2):
        _, out["load_host_then_upload_s"] = timed(
            lambda: load_records(p, pin=True).records.device_tensors())
    ok = all(torch.equal(v, back.records.device_tensors()[k])
             for k, v in t.records.device_tensors().items())
    out["round_trip_equal"] = ok
    out["device_load_GBps"] = out["file_bytes"] / out["load_device_s"] / 1e9
    print(json.dumps(out))
    os.remove(p)


if __name__ == "__main__":
    main()

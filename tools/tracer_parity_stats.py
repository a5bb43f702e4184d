"""How close the device tracer is to the reference's records on the golden
scenes: paths whose record count differs, and per field the share of values
that are bit-identical and the largest relative difference (diagnostic for
tests/test_gpu_tracer.py's bars)."""
import json
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np  # noqa: E402

from conftest import golden  # noqa: E402
from oracle import pathgraph_oracle as O  # noqa: E402
from test_gpu_tracer import INT, TRACE_CASES, VEC, _trace  # noqa: E402

out = {}
for name in TRACE_CASES:
    z = golden(name)
    _, _, t = _trace(name)
    ref_rec, ref_paths = O.load_golden_records(z)
    cnt, rc = t.paths.rec_count, ref_paths["rec_count"]
    same = cnt == rc
    rows = np.concatenate([np.arange(s, s + c) for s, c in zip(t.paths.rec_start[same], cnt[same])])
    rrows = np.concatenate([np.arange(s, s + c) for s, c in zip(ref_paths["rec_start"][same], rc[same])])
    st = {"paths": int(cnt.size), "paths_differing_in_length": int((~same).sum()),
          "records_compared": int(rows.size)}
    for f in VEC + INT:
        a, b = getattr(t.records, f)[rows], ref_rec[f][rrows]
        eq = (a == b) if a.dtype.kind != "f" else ((a == b) | (np.isnan(a) & np.isnan(b)))
        eq = eq.reshape(len(rows), -1).all(axis=1)
        d = {"bit_identical": float(eq.mean())}
        if a.dtype.kind == "f":
            r = np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-300)
            d["max_rel"] = float(np.nanmax(r, initial=0))
        st[f] = d
    out[name] = st
print(json.dumps(out, indent=1))

# the scenes without reference goldens, against the C tracer oracle
from oracle import tracer_oracle as T  # noqa: E402
from test_gpu_tracer import ORACLE_CASES  # noqa: E402
from paper_2404_11894_b200.harness.config import RenderConfig  # noqa: E402
from paper_2404_11894_b200.transport import render_pt  # noqa: E402

out2 = {}
for name, (factory, spp, md, seed) in ORACLE_CASES.items():
    scene = factory()
    cfg = RenderConfig(spp=spp, max_depth=md, seed=seed)
    t = render_pt(scene, cfg, with_records=True)
    ref_rec, ref_paths = T.trace_records(scene, cfg)
    same = t.paths.rec_count == ref_paths["rec_count"]
    st = {"paths": int(same.size), "paths_differing_in_length": int((~same).sum())}
    if same.all():
        for f in VEC:
            a, b = getattr(t.records, f), ref_rec[f]
            r = np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-300)
            st[f] = float(np.nanmax(r, initial=0))
    out2[name] = st
print(json.dumps(out2, indent=1))

"""Diagnostic: rows whose fixed point moves between late iterations (K = 1)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2404_11894_b200 import scenes as S
from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.pathgraph import build_graph, solve
from paper_2404_11894_b200.transport import render_pt

cfg = RenderConfig(spp=2, max_depth=12, seed=5)
out = render_pt(S.scene_c1((12, 12), floor=True), cfg, with_records=True)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 1
g = build_graph(out, K, seed=0)
kind = out.records.kind
nxt = g.next_idx
from paper_2404_11894_b200.pathgraph import aggregate_direct, aggregate_indirect, propagate
for k in (0, 1, 2, 3):
    r0 = solve(g, iterations=k, tol=0.0)
    ik = np.array(r0.incoming)
    r1 = solve(g, iterations=k + 1, tol=0.0)
    want = propagate(g, aggregate_indirect(g, ik) + aggregate_direct(g))
    got = np.array(r1.incoming)
    bad = np.flatnonzero(np.any(np.abs(got - want) > 1e-4 * np.abs(want) + 1e-7, axis=1))
    ch = np.where(nxt[bad] >= 0, nxt[bad], -1)
    print(f"step {k}->{k+1}: {bad.size} rows off; kinds {np.bincount(kind[bad], minlength=2)}; "
          f"child kinds {np.bincount(kind[ch[ch >= 0]], minlength=2)}; rows {bad[:8]} children {ch[:8]}")
    if bad.size:
        print(got[bad[:3]], want[bad[:3]])

import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from conftest import golden
from test_gpu_graph import _trace_from_golden, CASES
from paper_2404_11894_b200.pathgraph import build_graph
def rel(a, b):
    a = np.asarray(a, float); b = np.asarray(b, float)
    return float((np.abs(a - b) / np.maximum(np.abs(b), 1e-300)).max())
for name, K in CASES:
    z = golden(name); t = _trace_from_golden(z); g = build_graph(t, K, seed=int(z["seed"])); p = f"K{K}_"
    print(name, K, "W %.2e" % rel(g.w_indirect.data, z[p + "w_data"]),
          " ".join("%s %.2e" % (a, rel(getattr(g, a), z[p + a])) for a in ("phat_ind", "phat_dir_phase", "phat_dir_emit")),
          "dbar %.2e" % rel(g.d_bar, z[p + "d_bar"]),
          "inc", all(np.array_equal(getattr(g, a), z[p + a]) for a in ("included_phase", "included_emit")))

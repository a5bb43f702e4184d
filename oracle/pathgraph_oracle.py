"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference's path graph.

Follows, function by function:
  next_index           transport/records.py:128-140
  cluster_points       pathgraph/clustering.py:28-148  (hash grid + brute fallback,
                       LIFO split loop, numbering); numpy's Generator is the
                       RNG, exactly as in the reference (graph.py:59-60)
  marginals            pathgraph/graph.py:94-120
  operators            pathgraph/graph.py:123-168 (W as scipy CSR, D-bar)
  solve                pathgraph/solve.py:41-98 + operators.py:17-47
  splat                pathgraph/solve.py:101-132
  dense_*              pathgraph/dense.py:25-85

The candidate search is vectorised over points (a sorted cell table probed
27 times) instead of the reference's per-cell Python loop, and groups come
from a stable argsort instead of one nonzero() per center; both give the same
result by construction (same candidate set, same fp64 rounding, same
lowest-index tie-breaking).  Pinned by tests/test_oracle.py against the
reference's own outputs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

INV_PI = 1.0 / np.pi
INV_4PI = 1.0 / (4.0 * np.pi)


# ------------------------------------------------------------ records
def next_index(path_idx: np.ndarray) -> np.ndarray:
    """child = r+1 when on the same path, else -1 (records.py:128-140)."""
    n = path_idx.shape[0]
    out = np.full(n, -1, dtype=np.int64)
    same = np.flatnonzero(path_idx[1:] == path_idx[:-1]) if n > 1 else np.zeros(0, np.int64)
    out[same] = same + 1
    return out


def class_keys(kind, class_id) -> np.ndarray:
    """graph.py:59"""
    return np.asarray(kind, np.int64) * (1 << 32) + np.asarray(class_id, np.int64)


# ---------------------------------------------------------- clustering
@dataclass
class Cluster:
    center: int
    members: np.ndarray


def _sq_dist(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """((dx*dx + dy*dy) + dz*dz) elementwise, numpy's rounding order."""
    d = a - b
    return (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]


def nearest_center(pts: np.ndarray, centers: np.ndarray) -> np.ndarray:
    """Exact nearest center, the reference's grid procedure (clustering.py:96-148)."""
    n, m = pts.shape[0], centers.shape[0]
    if m == 1:
        return np.zeros(n, dtype=np.int64)
    lo = pts.min(axis=0)
    extent = pts.max(axis=0) - lo
    volume = float(np.prod(np.maximum(extent, 1e-12)))
    cell = max((volume / m) ** (1.0 / 3.0), 1e-9)
    ccell = np.floor((centers - lo) / cell).astype(np.int64)
    pcell = np.floor((pts - lo) / cell).astype(np.int64)
    # cell table: centers sorted by a collision-free key over the padded box
    span = np.maximum(pcell.max(axis=0), ccell.max(axis=0)) + 3
    def key(c):
        return ((c[:, 0] + 1) * span[1] + (c[:, 1] + 1)) * span[2] + (c[:, 2] + 1)
    order = np.argsort(key(ccell), kind="stable")
    skeys = key(ccell)[order]
    best_d = np.full(n, np.inf)
    best_j = np.full(n, -1, dtype=np.int64)
    for off in np.array(np.meshgrid([-1, 0, 1], [-1, 0, 1], [-1, 0, 1], indexing="ij")).reshape(3, -1).T:
        nk = key(pcell + off)
        lo_i = np.searchsorted(skeys, nk, side="left")
        hi_i = np.searchsorted(skeys, nk, side="right")
        cnt = hi_i - lo_i
        for t in range(int(cnt.max(initial=0))):
            sel = np.flatnonzero(cnt > t)
            j = order[lo_i[sel] + t]
            d2 = _sq_dist(pts[sel], centers[j])
            better = (d2 < best_d[sel]) | ((d2 == best_d[sel]) & (j < best_j[sel]))
            best_d[sel[better]] = d2[better]
            best_j[sel[better]] = j[better]
    fallback = np.flatnonzero((best_j < 0) | ~(np.sqrt(best_d) < cell))
    for s in range(0, fallback.shape[0], 2048):
        chunk = fallback[s:s + 2048]
        d2 = _sq_dist(pts[chunk][:, None, :], centers[None, :, :])
        best_j[chunk] = np.argmin(d2, axis=1)
    return best_j


def nearest_center_per_cell(pts: np.ndarray, centers: np.ndarray) -> np.ndarray:
    """The same assignment as nearest_center, computed with the reference's own
    control structure (clustering.py:96-148): a Python loop over the occupied
    cells, the 27-cell candidate list per cell, brute force for the rest.
    Used where the reference's CPU COST is what is being measured (bench.py's
    reference arm); nearest_center is the fast checker."""
    n, m = pts.shape[0], centers.shape[0]
    if m == 1:
        return np.zeros(n, dtype=np.int64)
    lo = pts.min(axis=0)
    volume = float(np.prod(np.maximum(pts.max(axis=0) - lo, 1e-12)))
    cell = max((volume / m) ** (1.0 / 3.0), 1e-9)
    table: dict = {}
    for j, key in enumerate(map(tuple, np.floor((centers - lo) / cell).astype(np.int64))):
        table.setdefault(key, []).append(j)
    pc = np.floor((pts - lo) / cell).astype(np.int64)
    order = np.lexsort((pc[:, 2], pc[:, 1], pc[:, 0]))
    pcs = pc[order]
    cuts = np.concatenate(([0], np.flatnonzero(np.any(pcs[1:] != pcs[:-1], axis=1)) + 1, [n]))
    assign = np.full(n, -1, dtype=np.int64)
    rest = []
    for b, e in zip(cuts[:-1], cuts[1:]):
        rows = order[b:e]
        x, y, z = pcs[b]
        cand = sorted(j for dx in (-1, 0, 1) for dy in (-1, 0, 1) for dz in (-1, 0, 1)
                      for j in table.get((x + dx, y + dy, z + dz), ()))
        if not cand:
            rest.append(rows)
            continue
        cand = np.asarray(cand, dtype=np.int64)
        d2 = _sq_dist(pts[rows][:, None, :], centers[cand][None, :, :])
        k = np.argmin(d2, axis=1)
        assign[rows] = cand[k]
        far = np.sqrt(d2[np.arange(rows.shape[0]), k]) >= cell
        if far.any():
            rest.append(rows[far])
    if rest:
        rows = np.concatenate(rest)
        for s in range(0, rows.shape[0], 4096):
            chunk = rows[s:s + 4096]
            assign[chunk] = np.argmin(_sq_dist(pts[chunk][:, None, :], centers[None, :, :]), axis=1)
    return assign


def _split_loop(pts, groups, centers, K, rng):
    """LIFO split of groups larger than 2K (clustering.py:58-85)."""
    limit = 2 * K
    stack = [c for c, g in enumerate(groups) if g.shape[0] > limit]
    while stack:
        c = stack.pop()
        mem = groups[c]
        if mem.shape[0] <= limit:
            continue
        pool = mem[mem != centers[c]]
        if pool.shape[0] == 0:
            pool = mem
        newc = int(pool[rng.integers(pool.shape[0])])
        d_old = _sq_dist(pts[mem], pts[centers[c]][None, :])
        d_new = _sq_dist(pts[mem], pts[newc][None, :])
        go = d_new < d_old
        keep, moved = mem[~go], mem[go]
        if keep.shape[0] == 0 or moved.shape[0] == 0:
            h = mem.shape[0] // 2
            keep, moved = mem[:h], mem[h:]
        groups[c] = keep
        groups.append(moved)
        centers.append(newc)
        if keep.shape[0] > limit:
            stack.append(c)
        if moved.shape[0] > limit:
            stack.append(len(groups) - 1)


def cluster_points(positions, keys, K: int, rng: np.random.Generator, faithful: bool = False):
    """(cluster_id, [Cluster]) per compatibility class (clustering.py:28-93).

    faithful=True follows the reference's control structure and its cost
    (per-cell candidate loop, one nonzero() per center for the groups,
    clustering.py:54-55) -- same result."""
    if K < 1:
        raise ValueError("cluster size K must be >= 1")
    pos = np.asarray(positions, dtype=np.float64)
    keys = np.asarray(keys)
    cluster_id = np.full(pos.shape[0], -1, dtype=np.int64)
    clusters: list[Cluster] = []
    for key in np.unique(keys):
        rows = np.flatnonzero(keys == key)
        pts = pos[rows]
        n = rows.shape[0]
        m = (n + K - 1) // K
        picks = rng.choice(n, size=m, replace=False)
        if faithful:
            assign = nearest_center_per_cell(pts, pts[picks])
            groups = [np.flatnonzero(assign == c) for c in range(m)]
        else:
            assign = nearest_center(pts, pts[picks])
            order = np.argsort(assign, kind="stable")
            bounds = np.searchsorted(assign[order], np.arange(m + 1))
            groups = [order[bounds[c]:bounds[c + 1]] for c in range(m)]
        centers = [int(x) for x in picks]
        _split_loop(pts, groups, centers, K, rng)
        for g, c in zip(groups, centers):
            if g.shape[0] == 0:
                continue
            mem = np.sort(rows[g])
            cluster_id[mem] = len(clusters)
            clusters.append(Cluster(center=int(rows[c]), members=mem))
    return cluster_id, clusters


# ------------------------------------------------- marginals / operators
def hg_pdf(cos_theta, g):
    """phase.py:17-21"""
    g2 = g * g
    den = 1.0 + g2 - 2.0 * g * cos_theta
    return INV_4PI * (1.0 - g2) / (den * np.sqrt(den))


def _strategy_pdf(rec, mem: np.ndarray, volume: bool, dirs: np.ndarray) -> np.ndarray:
    """out[b, l, j] = member l's strategy density toward member j's direction."""
    if volume:
        axis = -rec["omega_out"][mem]
        cos = np.einsum("bld,bjd->blj", axis, dirs)
        return hg_pdf(cos, rec["g"][mem][:, :, None])
    cos = np.einsum("bld,bjd->blj", rec["normal"][mem], dirs)
    return np.maximum(0.0, cos) * INV_PI


@dataclass
class Graph:
    rec: dict
    paths: dict
    width: int
    height: int
    spp: int
    cluster_id: np.ndarray
    clusters: list
    next_idx: np.ndarray
    phat_ind: np.ndarray = None
    phat_dir_phase: np.ndarray = None
    phat_dir_emit: np.ndarray = None
    included_phase: np.ndarray = None
    included_emit: np.ndarray = None
    w: sp.csr_matrix = None
    d_bar: np.ndarray = None


def _by_shape(graph: Graph):
    """Clusters grouped by (size, kind): {(s, kind): (n_s, s) member matrix}."""
    bins: dict = {}
    for cl in graph.clusters:
        bins.setdefault((cl.members.shape[0], int(graph.rec["kind"][cl.members[0]])), []).append(cl.members)
    return {k: np.vstack(v) for k, v in bins.items()}


def build_graph(rec: dict, paths: dict, width, height, spp, K: int, seed: int = 0,
                faithful: bool = False) -> Graph:
    """graph.py:56-69 with graph.py:94-168."""
    rng = np.random.default_rng(np.random.SeedSequence([seed & 0xFFFFFFFF, 0xC1A5]))
    cid, clusters = cluster_points(rec["pos"], class_keys(rec["kind"], rec["class_id"]), K, rng,
                                   faithful)
    g = Graph(rec, paths, width, height, spp, cid, clusters, next_index(rec["path_idx"]))
    build_operators(g)
    return g


def build_operators(g: Graph) -> None:
    """graph.py:94-168 (compute_marginals + _build_operators) over g.clusters."""
    rec = g.rec
    n = rec["pos"].shape[0]
    g.phat_ind, g.phat_dir_phase, g.phat_dir_emit = np.zeros(n), np.zeros(n), np.zeros(n)
    bins = _by_shape(g)
    for (s, kind), mem in bins.items():
        ks = float(s)
        pd = _strategy_pdf(rec, mem, kind == 0, rec["phase_dir"][mem])
        pe = _strategy_pdf(rec, mem, kind == 0, rec["emit_dir"][mem])
        p_ind = pd.sum(axis=1)
        g.phat_ind[mem] = p_ind
        g.phat_dir_phase[mem] = p_ind + ks * rec["pdf_emit_at_phase"][mem]
        p_de = pe.sum(axis=1) + ks * rec["pdf_emit"][mem]
        p_de[rec["emit_delta"][mem].astype(bool)] = ks
        g.phat_dir_emit[mem] = p_de
    g.included_phase = np.isfinite(g.phat_ind) & (g.phat_ind > 0.0)
    g.included_emit = np.isfinite(g.phat_dir_emit) & (g.phat_dir_emit > 0.0)
    ok_dp = g.included_phase & np.isfinite(g.phat_dir_phase) & (g.phat_dir_phase > 0.0)

    def safe_inv(p, ok):
        return np.where(ok, 1.0 / np.where(ok, p, 1.0), 0.0)

    inv_ind = safe_inv(g.phat_ind, g.included_phase)
    inv_de = safe_inv(g.phat_dir_emit, g.included_emit)
    inv_dp = safe_inv(g.phat_dir_phase, ok_dp)
    rows, cols, vals = [], [], []
    g.d_bar = np.zeros((n, 3))
    for (s, kind), mem in bins.items():
        pd = _strategy_pdf(rec, mem, kind == 0, rec["phase_dir"][mem])
        pe = _strategy_pdf(rec, mem, kind == 0, rec["emit_dir"][mem])
        w = pd * inv_ind[mem][:, None, :]
        rows.append(np.repeat(mem, s, axis=1).ravel())
        cols.append(np.tile(mem, (1, s)).ravel())
        vals.append(w.ravel())
        we = pe * inv_de[mem][:, None, :]
        wp = pd * inv_dp[mem][:, None, :]
        direct = np.einsum("brj,bjc->brc", we, rec["d_emit"][mem]) + \
            np.einsum("brj,bjc->brc", wp, rec["d_phase"][mem])
        g.d_bar[mem.ravel()] = (rec["coeff"][mem] * direct).reshape(-1, 3)
    if rows:
        r, c, v = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    else:
        r = c = np.zeros(0, np.int64)
        v = np.zeros(0)
    g.w = sp.csr_matrix((v, (r, c)), shape=(n, n))
    g.w.sort_indices()


# --------------------------------------------------------------- solve
def own_indirect(g: Graph, incoming: np.ndarray) -> np.ndarray:
    """solve.py:41-51"""
    rec = g.rec
    if rec["pos"].shape[0] == 0:
        return np.zeros((0, 3))
    cos = np.einsum("nd,nd->n", -rec["omega_out"], rec["phase_dir"])
    rho_v = hg_pdf(cos, rec["g"])
    rho_s = np.maximum(0.0, np.einsum("nd,nd->n", rec["normal"], rec["phase_dir"])) / np.pi
    rho = np.where(rec["kind"] == 0, rho_v, rho_s)
    pp = rec["pdf_phase"]
    ratio = np.where(pp > 0.0, rho / np.where(pp > 0.0, pp, 1.0), 0.0)
    return rec["coeff"] * ratio[:, None] * incoming


def aggregate_indirect(g: Graph, incoming):
    """operators.py:17-19"""
    return g.rec["coeff"] * (g.w @ incoming)


def propagate_linear(g: Graph, l_bar):
    """operators.py:41-47"""
    out = np.zeros_like(l_bar)
    has = g.next_idx >= 0
    ch = g.next_idx[has]
    out[has] = g.rec["w_cont"][ch] * l_bar[ch]
    return out


def propagate(g: Graph, l_bar):
    """operators.py:27-38"""
    out = g.rec["i_pt"].copy()
    has = g.next_idx >= 0
    ch = g.next_idx[has]
    out[has] = g.rec["w_cont"][ch] * l_bar[ch]
    return out


def residual_norm(new, old) -> float:
    """solve.py:54-61"""
    worst = 0.0
    for c in range(3):
        scale = max(float(np.max(np.abs(new[:, c]), initial=0.0)), 1e-12)
        worst = max(worst, float(np.max(np.abs(new[:, c] - old[:, c]), initial=0.0)) / scale)
    return worst


class Divergence(RuntimeError):
    pass


def solve(g: Graph, iterations: int = 10, tol: float = 1e-3):
    """solve.py:64-98 -> (incoming, i_bar, residuals, performed)."""
    term = (g.next_idx < 0)[:, None]
    base = propagate_linear(g, g.d_bar) + np.where(term, g.rec["i_pt"], 0.0)
    incoming = g.rec["i_pt"].copy()
    i_bar = own_indirect(g, incoming)
    residuals, grow = [], 0
    for _ in range(iterations):
        i_bar = aggregate_indirect(g, incoming)
        new = propagate_linear(g, i_bar) + base
        res = residual_norm(new, incoming)
        residuals.append(res)
        incoming = new
        if len(residuals) >= 2 and res > residuals[-2]:
            grow += 1
            if grow >= 3:
                raise Divergence(residuals)
        else:
            grow = 0
        if res < tol:
            break
    return incoming, i_bar, residuals, len(residuals)


def splat(g: Graph, i_bar, mode: str = "pt", d_bar=None) -> np.ndarray:
    """solve.py:101-132; mode in {"pt", "extra", "aggregated"}."""
    p = g.paths
    vals = p["d_cam"].copy()
    has = p["rec_count"] > 0
    r0 = p["rec_start"][has]
    direct = {"pt": lambda: p["direct0"][has], "extra": lambda: p["extra_direct"][has],
              "aggregated": lambda: (g.d_bar if d_bar is None else d_bar)[r0]}[mode]()
    vals[has] += p["cam_weight"][has] * (direct + i_bar[r0])
    per = vals.reshape(g.width * g.height, g.spp, 3)
    acc = np.zeros((g.width * g.height, 3))
    for s in range(g.spp):
        acc += per[:, s]
    return (acc / g.spp).reshape(g.height, g.width, 3)


def splat_pt(paths: dict, width, height, spp) -> np.ndarray:
    """records.py:259-265"""
    est = paths["pt_estimate"].reshape(width * height, spp, 3)
    acc = np.zeros((width * height, 3))
    for s in range(spp):
        acc += est[:, s]
    return (acc / spp).reshape(height, width, 3)


# --------------------------------------------------------- dense oracle
def _rho(rec, row, d):
    if rec["kind"][row] == 0:
        return float(hg_pdf(float(-rec["omega_out"][row] @ d), rec["g"][row]))
    return max(0.0, float(rec["normal"][row] @ d)) * INV_PI


def dense_solve(g: Graph, iterations: int):
    """Explicit A+ (3,N,N), Ao (3,N,2N), P (3,N,N) iteration (dense.py:25-85)."""
    rec = g.rec
    n = rec["pos"].shape[0]
    ap = np.zeros((3, n, n))
    ao = np.zeros((3, n, 2 * n))
    pm = np.zeros((3, n, n))
    for cl in g.clusters:
        for a in cl.members:
            for b in cl.members:
                if g.included_phase[b]:
                    ap[:, a, b] = rec["coeff"][a] * (_rho(rec, a, rec["phase_dir"][b]) / g.phat_ind[b])
                if g.included_emit[b]:
                    ao[:, a, 2 * b] = rec["coeff"][a] * (_rho(rec, a, rec["emit_dir"][b]) / g.phat_dir_emit[b])
                if g.included_phase[b] and g.phat_dir_phase[b] > 0.0:
                    ao[:, a, 2 * b + 1] = rec["coeff"][a] * (_rho(rec, a, rec["phase_dir"][b]) / g.phat_dir_phase[b])
    for row in range(n):
        ch = g.next_idx[row]
        if ch >= 0:
            pm[:, row, ch] = rec["w_cont"][ch]
    light = np.zeros((3, 2 * n))
    light[:, 0::2] = rec["d_emit"].T
    light[:, 1::2] = rec["d_phase"].T
    term = g.next_idx < 0
    inc = rec["i_pt"].T.copy()
    ib = np.zeros((3, n))
    const = np.stack([pm[c] @ (ao[c] @ light[c]) for c in range(3)])
    for _ in range(iterations):
        ib = np.stack([ap[c] @ inc[c] for c in range(3)])
        inc = np.stack([pm[c] @ ib[c] for c in range(3)]) + const
        inc[:, term] = rec["i_pt"].T[:, term]
    return inc.T.copy(), ib.T.copy()


def load_golden_records(z) -> tuple[dict, dict]:
    """Split a golden .npz into record and path dicts."""
    rec = {k[4:]: z[k] for k in z.files if k.startswith("rec_")}
    paths = {k[5:]: z[k] for k in z.files if k.startswith("path_")}
    return rec, paths

/* TEST INFRASTRUCTURE ONLY -- C restatement of the reference's path-graph
 * build, for parity checks at the benchmarked sizes (millions of records),
 * where oracle/pathgraph_oracle.py (numpy) is too slow.  Nothing in the
 * product links this; tests/, smoke() and bench.py's CPU legs load it through
 * oracle/graph_oracle.py.
 *
 * Restates, under /root/reference/pkg/src/volpg:
 *   cluster_points      pathgraph/clustering.py:28-44   (classes in ascending key
 *                                                        order, one shared RNG)
 *   _cluster_class      pathgraph/clustering.py:47-93   (choice, assignment,
 *                                                        groups, LIFO split loop,
 *                                                        numbering)
 *   _nearest_center     pathgraph/clustering.py:96-148  (lo/extent/cell, the
 *                                                        27-cell candidate argmin,
 *                                                        brute-force fallback)
 *   compute_marginals   pathgraph/graph.py:94-120
 *   _build_operators    pathgraph/graph.py:123-168      (W blocks, D-bar)
 *   aggregate_indirect  pathgraph/operators.py:17-19    (coeff * (W @ v))
 * and, from numpy 2.x (the reference's RNG, graph.py:60; not vendored):
 *   PCG64 (XSL-RR 128/64), Generator.choice(n, m, replace=False) (tail
 *   shuffle for n > 10000 and m > n // 50, else Floyd + shuffle) and
 *   Generator.integers(k), both over Lemire's bounded draw with the bit
 *   generator's buffered 32-bit half.
 *
 * The brute-force fallback (clustering.py:142-147: global argmin, lowest
 * index on ties) is evaluated with a k-d tree whose pruning bound carries a
 * relative slack far above fp64 rounding, so every center that could tie is
 * still visited: the same answer as the full scan.
 *
 * fp64 arithmetic follows numpy's order: squared distances
 * ((dx*dx + dy*dy) + dz*dz), dot products ((a0*b0 + a1*b1) + a2*b2), sums
 * over cluster members in ascending member order.  Built with
 * -ffp-contract=off (no fused multiply-add).  Parallel loops run on pthreads
 * (og_set_threads; default: all online cores).
 */
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>


/* ------------------------------------------------------- parallel for */
#include <unistd.h>
static int g_threads = 0;
void og_set_threads(int t) { g_threads = t; }
static int n_threads(void) {
  if (g_threads > 0) return g_threads;
  long c = sysconf(_SC_NPROCESSORS_ONLN);
  return c > 0 ? (int)c : 1;
}
typedef void (*range_fn)(void* ctx, int64_t b, int64_t e);
typedef struct {
  range_fn fn;
  void* ctx;
  int64_t n, chunk;
  atomic_llong next;
} par_job;
static void* par_worker(void* arg) {
  par_job* j = (par_job*)arg;
  for (;;) {
    const int64_t b = atomic_fetch_add(&j->next, j->chunk);
    if (b >= j->n) break;
    j->fn(j->ctx, b, b + j->chunk < j->n ? b + j->chunk : j->n);
  }
  return NULL;
}
/* fn over [0, n) in chunks, dynamically scheduled over the threads */
static void par_for(int64_t n, int64_t chunk, range_fn fn, void* ctx) {
  if (n <= 0) return;
  par_job j;
  j.fn = fn;
  j.ctx = ctx;
  j.n = n;
  j.chunk = chunk > 0 ? chunk : 1;
  atomic_init(&j.next, 0);
  int t = n_threads();
  if ((int64_t)t > (n + j.chunk - 1) / j.chunk) t = (int)((n + j.chunk - 1) / j.chunk);
  pthread_t th[256];
  if (t > 256) t = 256;
  for (int i = 1; i < t; ++i) pthread_create(&th[i], NULL, par_worker, &j);
  par_worker(&j);
  for (int i = 1; i < t; ++i) pthread_join(th[i], NULL);
}

/* ------------------------------------------------------------------ RNG */
typedef struct {
  uint64_t s_hi, s_lo, i_hi, i_lo;
  int32_t has_u32;
  uint32_t u32;
} og_pcg;

static uint64_t pcg_next64(og_pcg* r) {
  const __uint128_t mult = ((__uint128_t)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
  __uint128_t st = ((__uint128_t)r->s_hi << 64) | r->s_lo;
  const __uint128_t inc = ((__uint128_t)r->i_hi << 64) | r->i_lo;
  st = st * mult + inc;
  r->s_hi = (uint64_t)(st >> 64);
  r->s_lo = (uint64_t)st;
  const uint64_t x = r->s_hi ^ r->s_lo;
  const unsigned rot = (unsigned)(r->s_hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

static uint32_t pcg_next32(og_pcg* r) {
  if (r->has_u32) {
    r->has_u32 = 0;
    return r->u32;
  }
  const uint64_t v = pcg_next64(r);
  r->has_u32 = 1;
  r->u32 = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

/* numpy random_bounded_uint64(state, 0, rng, 0, use_masked = 0) */
static uint64_t bounded(og_pcg* r, uint64_t rng) {
  if (rng == 0) return 0;
  if (rng <= 0xFFFFFFFFULL) {
    if (rng == 0xFFFFFFFFULL) return pcg_next32(r);
    const uint32_t excl = (uint32_t)rng + 1u;
    uint64_t m = (uint64_t)pcg_next32(r) * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      const uint32_t thr = (uint32_t)(0xFFFFFFFFu - (uint32_t)rng) % excl;
      while (left < thr) {
        m = (uint64_t)pcg_next32(r) * excl;
        left = (uint32_t)m;
      }
    }
    return m >> 32;
  }
  if (rng == 0xFFFFFFFFFFFFFFFFULL) return pcg_next64(r);
  const uint64_t excl = rng + 1;
  __uint128_t m = (__uint128_t)pcg_next64(r) * excl;
  uint64_t left = (uint64_t)m;
  if (left < excl) {
    const uint64_t thr = (0xFFFFFFFFFFFFFFFFULL - rng) % excl;
    while (left < thr) {
      m = (__uint128_t)pcg_next64(r) * excl;
      left = (uint64_t)m;
    }
  }
  return (uint64_t)(m >> 64);
}

/* Generator.integers(k) for k >= 1 */
int64_t og_rng_integers(og_pcg* r, int64_t k) { return (int64_t)bounded(r, (uint64_t)(k - 1)); }

/* Generator.choice(n, m, replace=False) -> out[m]; 0 ok, -1 bad arguments */
int og_rng_choice(og_pcg* r, int64_t n, int64_t m, int64_t* out) {
  if (m < 0 || m > n) return -1;
  if (n > 10000 && m > n / 50) {
    int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    if (!idx) return -2;
    for (int64_t i = 0; i < n; ++i) idx[i] = i;
    const int64_t first = (n - m) > 1 ? (n - m) : 1;
    for (int64_t i = n - 1; i >= first; --i) {
      const int64_t j = (int64_t)bounded(r, (uint64_t)i);
      const int64_t t = idx[j];
      idx[j] = idx[i];
      idx[i] = t;
    }
    memcpy(out, idx + (n - m), sizeof(int64_t) * (size_t)m);
    free(idx);
    return 0;
  }
  /* Floyd: val = bounded(j); if val was already chosen, take j */
  uint8_t* seen = (uint8_t*)calloc((size_t)(n / 8 + 1), 1);
  if (!seen) return -2;
  for (int64_t j = n - m; j < n; ++j) {
    int64_t v = (int64_t)bounded(r, (uint64_t)j);
    if (seen[v >> 3] & (1u << (v & 7))) v = j;
    seen[v >> 3] |= (uint8_t)(1u << (v & 7));
    out[j - (n - m)] = v;
  }
  free(seen);
  for (int64_t i = m - 1; i >= 1; --i) {
    const int64_t j = (int64_t)bounded(r, (uint64_t)i);
    const int64_t t = out[j];
    out[j] = out[i];
    out[i] = t;
  }
  return 0;
}

/* ------------------------------------------------------------ sorting */
/* stable LSD radix sort of (key, val) pairs by key over `bits` low bits */
static int radix_sort_pairs(uint64_t* key, int64_t* val, int64_t n, int bits) {
  if (n <= 1) return 0;
  uint64_t* k2 = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
  int64_t* v2 = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * 65536);
  if (!k2 || !v2 || !cnt) {
    free(k2); free(v2); free(cnt);
    return -2;
  }
  uint64_t *ks = key, *kd = k2;
  int64_t *vs = val, *vd = v2;
  for (int sh = 0; sh < bits; sh += 16) {
    memset(cnt, 0, sizeof(int64_t) * 65536);
    for (int64_t i = 0; i < n; ++i) cnt[(ks[i] >> sh) & 0xFFFF]++;
    int64_t acc = 0;
    for (int b = 0; b < 65536; ++b) {
      const int64_t c = cnt[b];
      cnt[b] = acc;
      acc += c;
    }
    for (int64_t i = 0; i < n; ++i) {
      const int64_t d = cnt[(ks[i] >> sh) & 0xFFFF]++;
      kd[d] = ks[i];
      vd[d] = vs[i];
    }
    uint64_t* tk = ks; ks = kd; kd = tk;
    int64_t* tv = vs; vs = vd; vd = tv;
  }
  if (ks != key) {
    memcpy(key, ks, sizeof(uint64_t) * (size_t)n);
    memcpy(val, vs, sizeof(int64_t) * (size_t)n);
  }
  free(k2); free(v2); free(cnt);
  return 0;
}

static int bits_for(uint64_t v) {
  int b = 0;
  while (b < 64 && (v >> b)) ++b;
  return b ? b : 1;
}

/* --------------------------------------------------------- distances */
static inline double sq_dist(const double* a, const double* b) {
  const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return (dx * dx + dy * dy) + dz * dz;
}

/* ------------------------------------------------------ k-d tree (fallback) */
typedef struct {
  double lo[3], hi[3];
  int64_t b, e;       /* leaf: center ids idx[b..e) */
  int64_t left, right; /* children, -1 for a leaf */
} kd_node;

typedef struct {
  kd_node* nodes;
  int64_t n_nodes, cap;
  int64_t* idx;
  const double* c;
} kd_tree;

static int cmp_axis;
static const double* cmp_c;
static int cmp_ids(const void* a, const void* b) {
  const double x = cmp_c[*(const int64_t*)a * 3 + cmp_axis];
  const double y = cmp_c[*(const int64_t*)b * 3 + cmp_axis];
  return (x > y) - (x < y);
}

static int64_t kd_build(kd_tree* t, int64_t b, int64_t e) {
  if (t->n_nodes == t->cap) {
    t->cap = t->cap ? t->cap * 2 : 1024;
    t->nodes = (kd_node*)realloc(t->nodes, sizeof(kd_node) * (size_t)t->cap);
  }
  const int64_t id = t->n_nodes++;
  kd_node nd;
  for (int a = 0; a < 3; ++a) {
    nd.lo[a] = INFINITY;
    nd.hi[a] = -INFINITY;
  }
  for (int64_t i = b; i < e; ++i)
    for (int a = 0; a < 3; ++a) {
      const double v = t->c[t->idx[i] * 3 + a];
      if (v < nd.lo[a]) nd.lo[a] = v;
      if (v > nd.hi[a]) nd.hi[a] = v;
    }
  nd.b = b;
  nd.e = e;
  nd.left = nd.right = -1;
  if (e - b > 16) {
    int ax = 0;
    for (int a = 1; a < 3; ++a)
      if (nd.hi[a] - nd.lo[a] > nd.hi[ax] - nd.lo[ax]) ax = a;
    cmp_axis = ax;
    cmp_c = t->c;
    qsort(t->idx + b, (size_t)(e - b), sizeof(int64_t), cmp_ids);
    const int64_t mid = b + (e - b) / 2;
    const int64_t l = kd_build(t, b, mid);
    const int64_t r = kd_build(t, mid, e);
    nd.left = l;
    nd.right = r;
  }
  t->nodes[id] = nd;
  return id;
}

static inline double box_lb(const kd_node* nd, const double* p) {
  double s = 0.0;
  for (int a = 0; a < 3; ++a) {
    double d = 0.0;
    if (p[a] < nd->lo[a]) d = nd->lo[a] - p[a];
    else if (p[a] > nd->hi[a]) d = p[a] - nd->hi[a];
    s += d * d;
  }
  return s;
}

/* global argmin of sq_dist over all centers, lowest index on ties */
static int64_t kd_nearest(const kd_tree* t, const double* p) {
  double best = INFINITY;
  int64_t bj = -1;
  int64_t stack[256];
  int sp = 0;
  stack[sp++] = 0;
  while (sp) {
    const kd_node* nd = &t->nodes[stack[--sp]];
    if (box_lb(nd, p) * (1.0 - 1e-9) > best) continue;
    if (nd->left < 0) {
      for (int64_t i = nd->b; i < nd->e; ++i) {
        const int64_t j = t->idx[i];
        const double d2 = sq_dist(p, t->c + j * 3);
        if (d2 < best || (d2 == best && j < bj)) {
          best = d2;
          bj = j;
        }
      }
      continue;
    }
    const kd_node* L = &t->nodes[nd->left];
    const kd_node* R = &t->nodes[nd->right];
    const double dl = box_lb(L, p), dr = box_lb(R, p);
    if (dl <= dr) {
      stack[sp++] = nd->right;
      stack[sp++] = nd->left;
    } else {
      stack[sp++] = nd->left;
      stack[sp++] = nd->right;
    }
  }
  return bj;
}

/* ------------------------------------------------- nearest center (:96-148) */
typedef struct {
  int64_t cx, cy, cz;
  int64_t start, count; /* run in the center order */
  int used;
} cell_slot;

static inline uint64_t cell_hash(int64_t x, int64_t y, int64_t z) {
  uint64_t h = (uint64_t)x * 0x9E3779B97F4A7C15ULL;
  h ^= (uint64_t)y * 0xC2B2AE3D27D4EB4FULL + (h << 6) + (h >> 2);
  h ^= (uint64_t)z * 0x165667B19E3779F9ULL + (h << 6) + (h >> 2);
  h ^= h >> 31;
  return h * 0xD6E8FEB86659FD93ULL;
}

static const cell_slot* cell_find(const cell_slot* tab, uint64_t mask, int64_t x, int64_t y,
                                  int64_t z) {
  uint64_t h = cell_hash(x, y, z) & mask;
  while (tab[h].used) {
    if (tab[h].cx == x && tab[h].cy == y && tab[h].cz == z) return &tab[h];
    h = (h + 1) & mask;
  }
  return NULL;
}

typedef struct {
  const double *pts, *cen;
  const int64_t *pcell, *pid, *run;
  const cell_slot* tab;
  uint64_t mask;
  const int64_t* corder;
  double cell;
  int64_t* assign;
  uint8_t* far;
  const kd_tree* tree;
} assign_ctx;

/* the 27-cell candidate argmin of every point in runs [b, e) (:121-140) */
static void assign_runs(void* vctx, int64_t b, int64_t e) {
  const assign_ctx* c = (const assign_ctx*)vctx;
  int64_t ccap = 1024;
  int64_t* cand = (int64_t*)malloc(sizeof(int64_t) * (size_t)ccap);
  for (int64_t r = b; r < e; ++r) {
    /* a hashed run may mix cells: the candidates are gathered again
     * whenever the cell changes */
    int64_t lx = INT64_MIN, ly = 0, lz = 0, nc = 0;
    for (int64_t ii = c->run[r]; ii < c->run[r + 1]; ++ii) {
      const int64_t i = c->pid[ii];
      const int64_t x = c->pcell[i * 3], y = c->pcell[i * 3 + 1], z = c->pcell[i * 3 + 2];
      if (x != lx || y != ly || z != lz) {
      lx = x;
      ly = y;
      lz = z;
      nc = 0;
      for (int dx = -1; dx <= 1; ++dx)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dz = -1; dz <= 1; ++dz) {
            const cell_slot* sl = cell_find(c->tab, c->mask, x + dx, y + dy, z + dz);
            if (!sl) continue;
            if (nc + sl->count > ccap) {
              while (nc + sl->count > ccap) ccap *= 2;
              cand = (int64_t*)realloc(cand, sizeof(int64_t) * (size_t)ccap);
            }
            for (int64_t k = 0; k < sl->count; ++k) cand[nc++] = c->corder[sl->start + k];
          }
      }
      if (!nc) {
        c->far[i] = 1; /* no center in the neighbourhood (:129-131) */
        continue;
      }
      double best = INFINITY;
      int64_t bj = -1;
      for (int64_t k = 0; k < nc; ++k) {
        const int64_t j = cand[k];
        const double d2 = sq_dist(c->pts + i * 3, c->cen + j * 3);
        if (bj < 0 || d2 < best || (d2 == best && j < bj)) { /* argmin over sorted ids */
          best = d2;
          bj = j;
        }
      }
      c->assign[i] = bj;
      if (sqrt(best) >= c->cell) c->far[i] = 1; /* too_far (:138-140) */
    }
  }
  free(cand);
}

/* brute-force rows (:142-147) */
static void assign_far(void* vctx, int64_t b, int64_t e) {
  const assign_ctx* c = (const assign_ctx*)vctx;
  for (int64_t i = b; i < e; ++i)
    if (c->far[i]) c->assign[i] = kd_nearest(c->tree, c->pts + i * 3);
}

/* assign[i] = nearest center of pts[i]; returns the fallback count, < 0 on error */
static int64_t nearest_center(const double* pts, int64_t n, const double* cen, int64_t m,
                              int64_t* assign) {
  if (n <= 0 || m <= 0) return 0;
  if (m == 1) {
    for (int64_t i = 0; i < n; ++i) assign[i] = 0;
    return 0;
  }
  double lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    lo[a] = INFINITY;
    hi[a] = -INFINITY;
  }
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      const double v = pts[i * 3 + a];
      if (v < lo[a]) lo[a] = v;
      if (v > hi[a]) hi[a] = v;
    }
  double ext[3];
  for (int a = 0; a < 3; ++a) {
    ext[a] = hi[a] - lo[a];
    if (!(ext[a] >= 1e-12)) ext[a] = 1e-12; /* np.maximum(extent, 1e-12) */
  }
  const double volume = (ext[0] * ext[1]) * ext[2];
  double cell = pow(volume / (double)m, 1.0 / 3.0);
  if (!(cell >= 1e-9)) cell = 1e-9;

  /* center cells, centers ordered by (cell, id) */
  int64_t* ccell = (int64_t*)malloc(sizeof(int64_t) * 3 * (size_t)m);
  int64_t* pcell = (int64_t*)malloc(sizeof(int64_t) * 3 * (size_t)n);
  for (int64_t i = 0; i < m; ++i)
    for (int a = 0; a < 3; ++a) ccell[i * 3 + a] = (int64_t)floor((cen[i * 3 + a] - lo[a]) / cell);
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) pcell[i * 3 + a] = (int64_t)floor((pts[i * 3 + a] - lo[a]) / cell);
  int64_t cmin[3], cmax[3];
  for (int a = 0; a < 3; ++a) {
    cmin[a] = INT64_MAX;
    cmax[a] = INT64_MIN;
  }
  for (int64_t i = 0; i < m; ++i)
    for (int a = 0; a < 3; ++a) {
      if (ccell[i * 3 + a] < cmin[a]) cmin[a] = ccell[i * 3 + a];
      if (ccell[i * 3 + a] > cmax[a]) cmax[a] = ccell[i * 3 + a];
    }
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      if (pcell[i * 3 + a] < cmin[a]) cmin[a] = pcell[i * 3 + a];
      if (pcell[i * 3 + a] > cmax[a]) cmax[a] = pcell[i * 3 + a];
    }
  int bx = bits_for((uint64_t)(cmax[0] - cmin[0] + 1)), by = bits_for((uint64_t)(cmax[1] - cmin[1] + 1)),
      bz = bits_for((uint64_t)(cmax[2] - cmin[2] + 1));
  const int packable = bx + by + bz <= 62;

  /* centers by cell (stable in id): a hash of runs */
  uint64_t* ck = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)m);
  int64_t* cid = (int64_t*)malloc(sizeof(int64_t) * (size_t)m);
  for (int64_t i = 0; i < m; ++i) {
    ck[i] = cell_hash(ccell[i * 3], ccell[i * 3 + 1], ccell[i * 3 + 2]);
    cid[i] = i;
  }
  radix_sort_pairs(ck, cid, m, 64); /* equal cells are equal hashes; collisions split below */
  uint64_t cap = 1;
  while (cap < (uint64_t)(2 * m + 2)) cap <<= 1;
  cell_slot* tab = (cell_slot*)calloc(cap, sizeof(cell_slot));
  int64_t* corder = (int64_t*)malloc(sizeof(int64_t) * (size_t)m);
  int64_t at = 0;
  for (int64_t b = 0; b < m;) {
    int64_t e = b + 1;
    while (e < m && ck[e] == ck[b]) ++e;
    /* one hash value may hold several cells (a collision): group them */
    for (int64_t i = b; i < e; ++i) {
      const int64_t j = cid[i];
      if (j < 0) continue;
      const int64_t x = ccell[j * 3], y = ccell[j * 3 + 1], z = ccell[j * 3 + 2];
      const int64_t start = at;
      for (int64_t k = i; k < e; ++k) {
        const int64_t q = cid[k];
        if (q >= 0 && ccell[q * 3] == x && ccell[q * 3 + 1] == y && ccell[q * 3 + 2] == z) {
          corder[at++] = q; /* ascending: the sort is stable in id */
          cid[k] = -1;
        }
      }
      uint64_t h = cell_hash(x, y, z) & (cap - 1);
      while (tab[h].used) h = (h + 1) & (cap - 1);
      tab[h].cx = x;
      tab[h].cy = y;
      tab[h].cz = z;
      tab[h].start = start;
      tab[h].count = at - start;
      tab[h].used = 1;
    }
    b = e;
  }
  free(ck);
  free(cid);

  /* points grouped by cell (the reference walks occupied cells) */
  uint64_t* pk = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
  int64_t* pid = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t x = pcell[i * 3] - cmin[0], y = pcell[i * 3 + 1] - cmin[1], z = pcell[i * 3 + 2] - cmin[2];
    pk[i] = packable ? (((uint64_t)x << (by + bz)) | ((uint64_t)y << bz) | (uint64_t)z)
                     : cell_hash(pcell[i * 3], pcell[i * 3 + 1], pcell[i * 3 + 2]);
    pid[i] = i;
  }
  radix_sort_pairs(pk, pid, n, packable ? (bx + by + bz) : 64);
  /* run starts */
  int64_t n_runs = 0;
  int64_t* run = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t i = 0; i < n; ++i)
    if (i == 0 || pk[i] != pk[i - 1]) run[n_runs++] = i;
  run[n_runs] = n;
  free(pk);

  uint8_t* far = (uint8_t*)calloc((size_t)n, 1);
  assign_ctx ac = {pts, cen, pcell, pid, run, tab, cap - 1, corder, cell, assign, far, NULL};
  par_for(n_runs, 64, assign_runs, &ac);
  int64_t n_far = 0;
  for (int64_t i = 0; i < n; ++i) n_far += far[i];
  if (n_far) {
    kd_tree t = {0};
    t.c = cen;
    t.idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)m);
    for (int64_t j = 0; j < m; ++j) t.idx[j] = j;
    kd_build(&t, 0, m);
    ac.tree = &t;
    par_for(n, 4096, assign_far, &ac);
    free(t.nodes);
    free(t.idx);
  }
  free(far);
  free(run);
  free(pid);
  free(tab);
  free(corder);
  free(ccell);
  free(pcell);
  return n_far;
}

/* --------------------------------------------------------- clustering */
typedef struct {
  int64_t b, len; /* segment of the class's member pool */
} seg;

/* cluster_points (clustering.py:28-93).  Outputs: cluster_id[n]; clusters in
 * the reference's order as center[M], member_off[M+1], members[n] (record
 * indices, ascending within a cluster).  center/member_off need room for n+1.
 * counts[0] = M, counts[1] = splits, counts[2] = fallback points. */
int og_cluster(const double* pos, const int64_t* keys, int64_t n, int32_t K, og_pcg* rng,
               int64_t* cluster_id, int64_t* center, int64_t* member_off, int64_t* members,
               int64_t* counts) {
  if (K < 1) return -1;
  counts[0] = counts[1] = counts[2] = 0;
  member_off[0] = 0;
  if (n == 0) return 0;
  /* classes in ascending key order, rows ascending */
  uint64_t* key = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
  int64_t* row = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    key[i] = (uint64_t)keys[i] ^ 0x8000000000000000ULL;
    row[i] = i;
  }
  radix_sort_pairs(key, row, n, 64);
  int64_t M = 0;
  for (int64_t cb = 0; cb < n;) {
    int64_t ce = cb + 1;
    while (ce < n && key[ce] == key[cb]) ++ce;
    const int64_t* rows = row + cb;
    const int64_t nc = ce - cb;
    const int64_t mc = (nc + K - 1) / K;
    double* pts = (double*)malloc(sizeof(double) * 3 * (size_t)nc);
    for (int64_t i = 0; i < nc; ++i) memcpy(pts + i * 3, pos + rows[i] * 3, sizeof(double) * 3);
    int64_t* pick = (int64_t*)malloc(sizeof(int64_t) * (size_t)mc);
    if (og_rng_choice(rng, nc, mc, pick)) return -2;
    double* cen = (double*)malloc(sizeof(double) * 3 * (size_t)mc);
    for (int64_t j = 0; j < mc; ++j) memcpy(cen + j * 3, pts + pick[j] * 3, sizeof(double) * 3);
    int64_t* assign = (int64_t*)malloc(sizeof(int64_t) * (size_t)nc);
    counts[2] += nearest_center(pts, nc, cen, mc, assign);
    /* groups: members ascending (clustering.py:55) */
    int64_t* start = (int64_t*)calloc((size_t)mc + 1, sizeof(int64_t));
    for (int64_t i = 0; i < nc; ++i) start[assign[i] + 1]++;
    for (int64_t j = 0; j < mc; ++j) start[j + 1] += start[j];
    int64_t* pool = (int64_t*)malloc(sizeof(int64_t) * (size_t)nc);
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)mc);
    memcpy(fill, start, sizeof(int64_t) * (size_t)mc);
    for (int64_t i = 0; i < nc; ++i) pool[fill[assign[i]]++] = i;
    free(fill);
    int64_t gcap = mc + 16, ng = mc;
    seg* groups = (seg*)malloc(sizeof(seg) * (size_t)gcap);
    int64_t* gcen = (int64_t*)malloc(sizeof(int64_t) * (size_t)gcap);
    for (int64_t j = 0; j < mc; ++j) {
      groups[j].b = start[j];
      groups[j].len = start[j + 1] - start[j];
      gcen[j] = pick[j];
    }
    free(start);
    /* LIFO split loop (clustering.py:58-85) */
    const int64_t limit = 2 * (int64_t)K;
    int64_t scap = 64, sp = 0;
    int64_t* stack = (int64_t*)malloc(sizeof(int64_t) * (size_t)scap);
    for (int64_t c = 0; c < ng; ++c)
      if (groups[c].len > limit) {
        if (sp == scap) stack = (int64_t*)realloc(stack, sizeof(int64_t) * (size_t)(scap *= 2));
        stack[sp++] = c;
      }
    int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(limit + 1));
    int64_t tcap = limit + 1;
    while (sp) {
      const int64_t c = stack[--sp];
      const int64_t b = groups[c].b, len = groups[c].len;
      if (len <= limit) continue;
      int64_t* mem = pool + b;
      int64_t n_cand = 0;
      for (int64_t i = 0; i < len; ++i) n_cand += mem[i] != gcen[c];
      int64_t newc;
      if (n_cand == 0) {
        newc = mem[og_rng_integers(rng, len)];
      } else {
        int64_t k = og_rng_integers(rng, n_cand);
        newc = -1;
        for (int64_t i = 0; i < len; ++i)
          if (mem[i] != gcen[c] && k-- == 0) {
            newc = mem[i];
            break;
          }
      }
      if (tcap < len) {
        tcap = len;
        tmp = (int64_t*)realloc(tmp, sizeof(int64_t) * (size_t)tcap);
      }
      const double* po = pts + gcen[c] * 3;
      const double* pn = pts + newc * 3;
      int64_t nk = 0, nm = 0;
      for (int64_t i = 0; i < len; ++i) {
        const double dold = sq_dist(pts + mem[i] * 3, po), dnew = sq_dist(pts + mem[i] * 3, pn);
        if (dnew < dold) tmp[nm++] = mem[i]; /* argmin over (old, new): ties stay */
        else mem[nk++] = mem[i];
      }
      if (nk == 0 || nm == 0) {
        /* coincident points: halves by position (:75-78); one side empty
         * means the stable partition left mem untouched */
        nk = len / 2;
        nm = len - nk;
      } else {
        memcpy(mem + nk, tmp, sizeof(int64_t) * (size_t)nm);
      }
      if (ng == gcap) {
        gcap *= 2;
        groups = (seg*)realloc(groups, sizeof(seg) * (size_t)gcap);
        gcen = (int64_t*)realloc(gcen, sizeof(int64_t) * (size_t)gcap);
      }
      groups[c].len = nk;
      groups[ng].b = b + nk;
      groups[ng].len = nm;
      gcen[ng] = newc;
      ++ng;
      counts[1]++;
      if (sp + 2 > scap) stack = (int64_t*)realloc(stack, sizeof(int64_t) * (size_t)(scap *= 2));
      if (nk > limit) stack[sp++] = c;
      if (nm > limit) stack[sp++] = ng - 1;
    }
    free(tmp);
    free(stack);
    /* numbering: groups in order, empty ones skipped (:87-93) */
    for (int64_t c = 0; c < ng; ++c) {
      if (!groups[c].len) continue;
      const int64_t off = member_off[M];
      for (int64_t i = 0; i < groups[c].len; ++i) {
        const int64_t r = rows[pool[groups[c].b + i]];
        members[off + i] = r;
        cluster_id[r] = M;
      }
      member_off[M + 1] = off + groups[c].len;
      center[M] = rows[gcen[c]];
      ++M;
    }
    free(groups);
    free(gcen);
    free(pool);
    free(assign);
    free(cen);
    free(pick);
    free(pts);
    cb = ce;
  }
  free(key);
  free(row);
  counts[0] = M;
  return 0;
}

/* ------------------------------------------------- marginals / operators */
#define INV_PI (1.0 / 3.14159265358979323846)
#define INV_4PI (1.0 / (4.0 * 3.14159265358979323846))

static inline double dot3(const double* a, const double* b) {
  return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

static inline double hg_pdf(double cs, double g) { /* phase.py:17-21 */
  const double g2 = g * g;
  const double den = 1.0 + g2 - 2.0 * g * cs;
  return INV_4PI * (1.0 - g2) / (den * sqrt(den));
}

/* member l's strategy density toward direction d (graph.py:82-91) */
static inline double strategy_pdf(int volume, const double* omega_out, const double* normal,
                                  const double* g, int64_t l, const double* d) {
  if (volume) {
    const double a[3] = {-omega_out[l * 3], -omega_out[l * 3 + 1], -omega_out[l * 3 + 2]};
    return hg_pdf(dot3(a, d), g[l]);
  }
  const double c = dot3(normal + l * 3, d);
  return (c > 0.0 ? c : 0.0) * INV_PI;
}

typedef struct {
  const double *omega_out, *normal, *g, *phase_dir, *emit_dir, *pdf_emit_at_phase, *pdf_emit,
      *coeff, *d_emit, *d_phase;
  const uint8_t *emit_delta, *kind;
} og_records;

typedef struct {
  const og_records* R;
  const int64_t *member_off, *members, *w_off;
  double *phat_ind, *phat_dir_phase, *phat_dir_emit, *w_blocks, *d_bar;
  uint8_t *inc_phase, *inc_emit;
} ops_ctx;

static void ops_range(void* vctx, int64_t b, int64_t e) {
  const ops_ctx* x = (const ops_ctx*)vctx;
  const og_records* R = x->R;
  int cap = 0;
  double *pd = NULL, *pe = NULL;
  for (int64_t c = b; c < e; ++c) {
    const int64_t* mem = x->members + x->member_off[c];
    const int s = (int)(x->member_off[c + 1] - x->member_off[c]);
    if (s > cap) {
      cap = s;
      pd = (double*)realloc(pd, sizeof(double) * (size_t)s * (size_t)s);
      pe = (double*)realloc(pe, sizeof(double) * (size_t)s * (size_t)s);
    }
    const int vol = R->kind[mem[0]] == 0;
    const double k = (double)s;
    /* pd[l][j] / pe[l][j]: member l's density at member j's direction (graph.py:82-91) */
    for (int l = 0; l < s; ++l)
      for (int j = 0; j < s; ++j) {
        pd[l * s + j] = strategy_pdf(vol, R->omega_out, R->normal, R->g, mem[l], R->phase_dir + mem[j] * 3);
        pe[l * s + j] = strategy_pdf(vol, R->omega_out, R->normal, R->g, mem[l], R->emit_dir + mem[j] * 3);
      }
    /* marginals (graph.py:107-120) */
    for (int j = 0; j < s; ++j) {
      double si = 0.0, se = 0.0;
      for (int l = 0; l < s; ++l) {
        si += pd[l * s + j];
        se += pe[l * s + j];
      }
      const int64_t r = mem[j];
      x->phat_ind[r] = si;
      x->phat_dir_phase[r] = si + k * R->pdf_emit_at_phase[r];
      x->phat_dir_emit[r] = R->emit_delta[r] ? k : se + k * R->pdf_emit[r];
      x->inc_phase[r] = isfinite(x->phat_ind[r]) && x->phat_ind[r] > 0.0;
      x->inc_emit[r] = isfinite(x->phat_dir_emit[r]) && x->phat_dir_emit[r] > 0.0;
    }
    /* W block and D-bar (graph.py:138-162) */
    for (int rr = 0; rr < s; ++rr) {
      const int64_t r = mem[rr];
      double acc[3] = {0.0, 0.0, 0.0}, acc2[3] = {0.0, 0.0, 0.0};
      for (int j = 0; j < s; ++j) {
        const int64_t q = mem[j];
        const double di = x->phat_ind[q], de = x->phat_dir_emit[q], dp = x->phat_dir_phase[q];
        const int okp = x->inc_phase[q];
        const int okdp = okp && isfinite(dp) && dp > 0.0;
        if (x->w_blocks)
          x->w_blocks[x->w_off[c] + (int64_t)rr * s + j] = okp ? pd[rr * s + j] / (di > 0 ? di : 1.0) : 0.0;
        const double we = x->inc_emit[q] ? pe[rr * s + j] / (de > 0 ? de : 1.0) : 0.0;
        const double wp = okdp ? pd[rr * s + j] / (dp > 0 ? dp : 1.0) : 0.0;
        for (int ch = 0; ch < 3; ++ch) {
          acc[ch] += we * R->d_emit[q * 3 + ch];
          acc2[ch] += wp * R->d_phase[q * 3 + ch];
        }
      }
      for (int ch = 0; ch < 3; ++ch) x->d_bar[r * 3 + ch] = R->coeff[r * 3 + ch] * (acc[ch] + acc2[ch]);
    }
  }
  free(pd);
  free(pe);
}

/* compute_marginals + _build_operators over the given clusters (member
 * lists ascending).  w_blocks (optional): cluster c's row-major s x s block
 * W[r][j] at w_off[c]. */
int og_operators(const og_records* R, int64_t M, const int64_t* member_off, const int64_t* members,
                 double* phat_ind, double* phat_dir_phase, double* phat_dir_emit, uint8_t* inc_phase,
                 uint8_t* inc_emit, const int64_t* w_off, double* w_blocks, double* d_bar) {
  ops_ctx x = {R, member_off, members, w_off, phat_ind, phat_dir_phase, phat_dir_emit,
               w_blocks, d_bar, inc_phase, inc_emit};
  par_for(M, 256, ops_range, &x);
  return 0;
}

typedef struct {
  const double* coeff;
  const int64_t *member_off, *members, *w_off;
  const double *w_blocks, *v;
  double* out;
} apply_ctx;

static void apply_range(void* vctx, int64_t b, int64_t e) {
  const apply_ctx* x = (const apply_ctx*)vctx;
  for (int64_t c = b; c < e; ++c) {
    const int64_t* mem = x->members + x->member_off[c];
    const int s = (int)(x->member_off[c + 1] - x->member_off[c]);
    const double* w = x->w_blocks + x->w_off[c];
    for (int rr = 0; rr < s; ++rr) {
      double acc[3] = {0.0, 0.0, 0.0};
      for (int j = 0; j < s; ++j)
        for (int ch = 0; ch < 3; ++ch) acc[ch] += w[(int64_t)rr * s + j] * x->v[mem[j] * 3 + ch];
      const int64_t r = mem[rr];
      for (int ch = 0; ch < 3; ++ch) x->out[r * 3 + ch] = x->coeff[r * 3 + ch] * acc[ch];
    }
  }
}

/* out = coeff * (W @ v) over the stored blocks (operators.py:17-19) */
int og_apply_w(const double* coeff, int64_t M, const int64_t* member_off, const int64_t* members,
               const int64_t* w_off, const double* w_blocks, const double* v, double* out) {
  apply_ctx x = {coeff, member_off, members, w_off, w_blocks, v, out};
  par_for(M, 512, apply_range, &x);
  return 0;
}

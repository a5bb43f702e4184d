/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference tracer.
 *
 * Follows /root/reference/pkg/src/volpg:
 *   rng.py:19-51 (splitmix64 streams), scenecore/geometry.py:18-174,
 *   scenecore/medium.py:33-214, scenecore/phase.py:17-70,
 *   scenecore/emitters.py:22-107, transport/kernels.py:40-553.
 * fp64, evaluation order as in the reference, built with -ffp-contract=off so
 * no multiply-add is fused (numba does not fuse either); with glibc's libm the
 * records match the reference's bit for bit (tests/test_oracle_tracer.py).
 * Used to generate the CPU reference arm's input records in bench.py and as
 * a second checker for the CUDA tracer; never linked into the product.
 */
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NO_HIT 1e30
#define T_EPS 1e-7
#define SURF_OFF 1e-6
#define MAXS 32
#define MAXE 16
#define MAXM 8

typedef struct {
  int ns, ne, nm, width, height;
  int stype[MAXS], mat[MAXS], emid[MAXS];
  double sp[MAXS][9], alb[MAXS][3];
  int etype[MAXE];
  double eval[MAXE][3], epos[MAXE][3], equad[MAXE][9], enrm[MAXE][3], earea[MAXE];
  int mkind[MAXM], dims[MAXM][3];
  double st[MAXM][3], ss[MAXM][3], mg[MAXM], mb[MAXM][6], mu[MAXM], mscale[MAXM];
  int64_t goff[MAXM];
  const float* grid;
  double cam[15];
} OScene;

typedef struct {
  double *pos, *omega_out, *normal, *coeff, *g, *phase_dir, *pdf_phase, *pdf_emit_at_phase,
      *emit_dir, *pdf_emit, *d_emit, *d_phase, *i_pt, *w_cont;
  uint8_t *kind, *emit_delta;
  int32_t* class_id;
  int64_t* path_idx;
  int32_t* depth;
} ORec;

typedef struct {
  double *cam_weight, *d_cam, *direct0, *direct0_nee, *direct0_phase, *pt_estimate;
} OPath;

static const double PI = 3.14159265358979323846;

/* ---------------------------------------------------------------- rng */
static uint64_t sm_next(uint64_t* s) {
  *s += 0x9E3779B97F4A7C15ull;
  uint64_t z = *s;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static double uni(uint64_t* s) { return (double)(sm_next(s) >> 11) * (1.0 / 9007199254740992.0); }
static uint64_t stream_for(int64_t seed, int64_t key, uint64_t salt) {
  uint64_t s = (uint64_t)seed ^ ((uint64_t)key * 0xD1342543DE82EF95ull);
  s += salt * 0x9E3779B97F4A7C15ull;
  uint64_t a = sm_next(&s), b = sm_next(&s);
  return a ^ (b >> 1);
}

static double pmax(double a, double b) { return b > a ? b : a; }
static double pmin(double a, double b) { return b < a ? b : a; }

/* ----------------------------------------------------------- geometry */
static void slab(const double* o, const double* d, const double* b, double* t0, double* t1) {
  *t0 = -NO_HIT;
  *t1 = NO_HIT;
  for (int a = 0; a < 3; ++a) {
    if (d[a] != 0.0) {
      double inv = 1.0 / d[a];
      double lo = (b[a] - o[a]) * inv, hi = (b[3 + a] - o[a]) * inv;
      if (lo > hi) { double t = lo; lo = hi; hi = t; }
      *t0 = pmax(*t0, lo);
      *t1 = pmin(*t1, hi);
    } else if (o[a] < b[a] || o[a] > b[3 + a]) {
      *t0 = 1.0;
      *t1 = -1.0;
      return;
    }
  }
}

static void qnormal(const double* u, const double* v, double* n) {
  double x = u[1] * v[2] - u[2] * v[1], y = u[2] * v[0] - u[0] * v[2], z = u[0] * v[1] - u[1] * v[0];
  double inv = 1.0 / sqrt(x * x + y * y + z * z);
  n[0] = x * inv; n[1] = y * inv; n[2] = z * inv;
}

static double hit_surface(const OScene* S, int i, const double* o, const double* d, double tmin) {
  const double* p = S->sp[i];
  if (S->stype[i] == 0) {
    double lx = o[0] - p[0], ly = o[1] - p[1], lz = o[2] - p[2];
    double b = lx * d[0] + ly * d[1] + lz * d[2];
    double c = lx * lx + ly * ly + lz * lz - p[3] * p[3];
    double disc = b * b - c;
    if (disc < 0.0) return NO_HIT;
    double s = sqrt(disc);
    if (-b - s > tmin) return -b - s;
    if (-b + s > tmin) return -b + s;
    return NO_HIT;
  }
  if (S->stype[i] == 1) {
    double t0, t1;
    slab(o, d, p, &t0, &t1);
    if (t0 > t1) return NO_HIT;
    if (t0 > tmin) return t0;
    if (t1 > tmin) return t1;
    return NO_HIT;
  }
  double n[3];
  qnormal(p + 3, p + 6, n);
  double den = d[0] * n[0] + d[1] * n[1] + d[2] * n[2];
  if (fabs(den) < 1e-12) return NO_HIT;
  double t = ((p[0] - o[0]) * n[0] + (p[1] - o[1]) * n[1] + (p[2] - o[2]) * n[2]) / den;
  if (t <= tmin) return NO_HIT;
  double hx = o[0] + t * d[0] - p[0], hy = o[1] + t * d[1] - p[1], hz = o[2] + t * d[2] - p[2];
  double uu = p[3] * p[3] + p[4] * p[4] + p[5] * p[5];
  double vv = p[6] * p[6] + p[7] * p[7] + p[8] * p[8];
  double a = (hx * p[3] + hy * p[4] + hz * p[5]) / uu;
  double bb = (hx * p[6] + hy * p[7] + hz * p[8]) / vv;
  if (a < 0.0 || a > 1.0 || bb < 0.0 || bb > 1.0) return NO_HIT;
  return t;
}

static double nearest(const OScene* S, const double* o, const double* d, double tmin, double tmax,
                      int* sid) {
  double best = tmax;
  *sid = -1;
  for (int i = 0; i < S->ns; ++i) {
    double t = hit_surface(S, i, o, d, tmin);
    if (t < best) { best = t; *sid = i; }
  }
  return best;
}

static void normal_at(const OScene* S, int i, const double* x, double* n) {
  const double* p = S->sp[i];
  if (S->stype[i] == 0) {
    double inv = 1.0 / p[3];
    n[0] = (x[0] - p[0]) * inv; n[1] = (x[1] - p[1]) * inv; n[2] = (x[2] - p[2]) * inv;
    return;
  }
  if (S->stype[i] == 1) {
    const double cand[6][3] = {{-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1}};
    const double dd[6] = {fabs(x[0] - p[0]), fabs(x[0] - p[3]), fabs(x[1] - p[1]),
                          fabs(x[1] - p[4]), fabs(x[2] - p[2]), fabs(x[2] - p[5])};
    int k = 0;
    double best = dd[0];
    for (int j = 1; j < 6; ++j)
      if (dd[j] < best) { best = dd[j]; k = j; }
    n[0] = cand[k][0]; n[1] = cand[k][1]; n[2] = cand[k][2];
    return;
  }
  qnormal(p + 3, p + 6, n);
}

/* ------------------------------------------------------------- media */
static double density(const OScene* S, int k, const double* x) {
  const double* b = S->mb[k];
  int nx = S->dims[k][0], ny = S->dims[k][1], nz = S->dims[k][2];
  long long ix = (long long)((x[0] - b[0]) / (b[3] - b[0]) * nx);
  long long iy = (long long)((x[1] - b[1]) / (b[4] - b[1]) * ny);
  long long iz = (long long)((x[2] - b[2]) / (b[5] - b[2]) * nz);
  if (ix < 0) ix = 0; if (ix > nx - 1) ix = nx - 1;
  if (iy < 0) iy = 0; if (iy > ny - 1) iy = ny - 1;
  if (iz < 0) iz = 0; if (iz > nz - 1) iz = nz - 1;
  return (double)S->grid[S->goff[k] + (iz * ny + iy) * nx + ix];
}

/* returns 1 if scattered; w = Tr/p */
static int fly_one(const OScene* S, int k, const double* o, const double* d, double a, double b,
                   uint64_t* rs, double* t_out, double* w) {
  const double* st = S->st[k];
  double len = b - a;
  w[0] = w[1] = w[2] = 1.0;
  *t_out = b;
  if (S->mkind[k] == 0) {
    double sb = (st[0] + st[1] + st[2]) / 3.0;
    if (sb <= 0.0) return 0;
    double u = uni(rs);
    double dist = -log1p(-u) / sb;
    if (dist >= len) {
      for (int c = 0; c < 3; ++c) w[c] = exp(-(st[c] - sb) * len);
      return 0;
    }
    for (int c = 0; c < 3; ++c) w[c] = exp(-(st[c] - sb) * dist) / sb;
    *t_out = a + dist;
    return 1;
  }
  double mu = S->mu[k];
  if (mu <= 0.0) return 0;
  double t = a;
  for (;;) {
    double u = uni(rs);
    t += -log1p(-u) / mu;
    if (t >= b) return 0;
    double x[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
    double dn = density(S, k, x) * S->mscale[k];
    double s0 = st[0] * dn, s1 = st[1] * dn, s2 = st[2] * dn;
    double sb = (s0 + s1 + s2) / 3.0;
    double u2 = uni(rs);
    if (u2 * mu < sb) {
      double inv = 1.0 / sb;
      for (int c = 0; c < 3; ++c) w[c] *= inv;
      *t_out = t;
      return 1;
    }
    double den = mu - sb;
    w[0] *= (mu - s0) / den;
    w[1] *= (mu - s1) / den;
    w[2] *= (mu - s2) / den;
  }
}

static void tr_one(const OScene* S, int k, const double* o, const double* d, double a, double b,
                   uint64_t* rs, double* w) {
  const double* st = S->st[k];
  double len = b - a;
  w[0] = w[1] = w[2] = 1.0;
  if (len <= 0.0) return;
  if (S->mkind[k] == 0) {
    for (int c = 0; c < 3; ++c) w[c] = exp(-st[c] * len);
    return;
  }
  double mu = S->mu[k];
  if (mu <= 0.0) return;
  double t = a;
  for (;;) {
    double u = uni(rs);
    t += -log1p(-u) / mu;
    if (t >= b) return;
    double x[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
    double dn = density(S, k, x) * S->mscale[k];
    for (int c = 0; c < 3; ++c) w[c] *= 1.0 - st[c] * dn / mu;
    if (w[0] == 0.0 && w[1] == 0.0 && w[2] == 0.0) return;
  }
}

static int fly(const OScene* S, const double* o, const double* d, double tlo, double thi,
               uint64_t* rs, double* t_out, int* mid, double* w) {
  double cur = tlo;
  w[0] = w[1] = w[2] = 1.0;
  *t_out = thi;
  *mid = -1;
  for (int it = 0; it < 2 * S->nm + 1; ++it) {
    int bk = -1;
    double ba = thi, bb = thi;
    for (int k = 0; k < S->nm; ++k) {
      double t0, t1;
      slab(o, d, S->mb[k], &t0, &t1);
      double a = pmax(t0, cur), b = pmin(t1, thi);
      if (b > a + 1e-12 && a < ba) { ba = a; bk = k; bb = b; }
    }
    if (bk < 0) return 0;
    double t, ww[3];
    int sc = fly_one(S, bk, o, d, ba, bb, rs, &t, ww);
    for (int c = 0; c < 3; ++c) w[c] *= ww[c];
    if (sc) { *t_out = t; *mid = bk; return 1; }
    cur = bb + 1e-12;
  }
  return 0;
}

static void transmit(const OScene* S, const double* o, const double* d, double tlo, double thi,
                     uint64_t* rs, double* w) {
  w[0] = w[1] = w[2] = 1.0;
  for (int k = 0; k < S->nm; ++k) {
    double t0, t1;
    slab(o, d, S->mb[k], &t0, &t1);
    double a = pmax(t0, tlo), b = pmin(t1, thi);
    if (b > a + 1e-12) {
      double tr[3];
      tr_one(S, k, o, d, a, b, rs, tr);
      for (int c = 0; c < 3; ++c) w[c] *= tr[c];
    }
  }
}

/* -------------------------------------------------------------- phase */
static double hg(double c, double g) {
  double g2 = g * g;
  double den = 1.0 + g2 - 2.0 * g * c;
  return (1.0 / (4.0 * PI)) * (1.0 - g2) / (den * sqrt(den));
}

static void frame(const double* n, double* t, double* s) {
  double bx = 1.0, by = 0.0, bz = 0.0;
  if (fabs(n[0]) > 0.9) { bx = 0.0; by = 1.0; }
  double tx = by * n[2] - bz * n[1], ty = bz * n[0] - bx * n[2], tz = bx * n[1] - by * n[0];
  double inv = 1.0 / sqrt(tx * tx + ty * ty + tz * tz);
  tx *= inv; ty *= inv; tz *= inv;
  t[0] = tx; t[1] = ty; t[2] = tz;
  s[0] = n[1] * tz - n[2] * ty;
  s[1] = n[2] * tx - n[0] * tz;
  s[2] = n[0] * ty - n[1] * tx;
}

static void around(const double* n, double a, double b, double c, double* out) {
  double t[3], s[3];
  frame(n, t, s);
  double dx = a * t[0] + b * s[0] + c * n[0];
  double dy = a * t[1] + b * s[1] + c * n[1];
  double dz = a * t[2] + b * s[2] + c * n[2];
  double inv = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
  out[0] = dx * inv; out[1] = dy * inv; out[2] = dz * inv;
}

static void hg_dir(double g, const double* ax, double u1, double u2, double* out) {
  double ct;
  if (fabs(g) < 1e-6) {
    ct = 1.0 - 2.0 * u1;
  } else {
    double s = (1.0 - g * g) / (1.0 - g + 2.0 * g * u1);
    ct = pmin(1.0, pmax(-1.0, (1.0 + g * g - s * s) / (2.0 * g)));
  }
  double st = sqrt(pmax(0.0, 1.0 - ct * ct));
  double phi = 2.0 * PI * u2;
  around(ax, st * cos(phi), st * sin(phi), ct, out);
}

static void cos_dir(const double* n, double u1, double u2, double* out) {
  double z = sqrt(pmax(1e-12, 1.0 - u2));
  double r = sqrt(pmax(0.0, u2));
  double phi = 2.0 * PI * u1;
  around(n, r * cos(phi), r * sin(phi), z, out);
}

/* ----------------------------------------------------------- emitters */
typedef struct {
  double w[3], pdf, rad[3];
  int delta;
} ESample;

static ESample nee(const OScene* S, const double* p, uint64_t* rs) {
  ESample o = {{0.0, 0.0, 1.0}, 1.0, {0.0, 0.0, 0.0}, 0};
  int ne = S->ne;
  double u = uni(rs);
  long long e = (long long)(u * ne);
  if (e > ne - 1) e = ne - 1;
  const double* val = S->eval[e];
  double sel = (double)ne;
  if (S->etype[e] == 1) {
    const double* q = S->equad[e];
    double u1 = uni(rs), u2 = uni(rs);
    double d[3];
    for (int a = 0; a < 3; ++a) d[a] = q[a] + u1 * q[3 + a] + u2 * q[6 + a] - p[a];
    double d2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
    if (d2 < 1e-16) return o;
    double dist = sqrt(d2);
    for (int a = 0; a < 3; ++a) o.w[a] = d[a] / dist;
    const double* nq = S->enrm[e];
    double cq = -(nq[0] * o.w[0] + nq[1] * o.w[1] + nq[2] * o.w[2]);
    o.pdf = d2 / (S->earea[e] * pmax(fabs(cq), 1e-12) * sel);
    if (cq <= 0.0) return o;
    double clear = dist - 1e-6 * pmax(1.0, dist);
    int sid;
    if (nearest(S, p, o.w, T_EPS, clear, &sid) < clear) return o;
    double tr[3];
    transmit(S, p, o.w, 0.0, dist, rs, tr);
    for (int c = 0; c < 3; ++c) o.rad[c] = val[c] * tr[c];
    return o;
  }
  o.delta = 1;
  if (S->etype[e] == 0) {
    double d[3];
    for (int a = 0; a < 3; ++a) d[a] = S->epos[e][a] - p[a];
    double d2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
    if (d2 < 1e-16) return o;
    double dist = sqrt(d2);
    for (int a = 0; a < 3; ++a) o.w[a] = d[a] / dist;
    double clear = dist - 1e-6 * pmax(1.0, dist);
    int sid;
    if (nearest(S, p, o.w, T_EPS, clear, &sid) < clear) return o;
    double tr[3];
    transmit(S, p, o.w, 0.0, dist, rs, tr);
    double inv = sel / d2;
    for (int c = 0; c < 3; ++c) o.rad[c] = val[c] * tr[c] * inv;
    return o;
  }
  for (int a = 0; a < 3; ++a) o.w[a] = -S->epos[e][a];
  int sid;
  if (nearest(S, p, o.w, T_EPS, NO_HIT, &sid) < NO_HIT) return o;
  double tr[3];
  transmit(S, p, o.w, 0.0, NO_HIT, rs, tr);
  for (int c = 0; c < 3; ++c) o.rad[c] = val[c] * tr[c] * sel;
  return o;
}

static double pdf_from_hit(const OScene* S, int sid, double t, const double* w) {
  if (sid < 0 || S->mat[sid] != 2) return 0.0;
  int e = S->emid[sid];
  if (S->etype[e] != 1) return 0.0;
  const double* nq = S->enrm[e];
  double c = fabs(nq[0] * w[0] + nq[1] * w[1] + nq[2] * w[2]);
  if (c < 1e-12) return 0.0;
  return t * t / (S->earea[e] * c * S->ne);
}

/* --------------------------------------------------- trace_one (fill=0/1) */
static int trace_path(const OScene* S, int64_t px, int64_t py, int64_t pid, int64_t seed,
                      int max_depth, int rr_start, double rr_floor, int fill, int64_t off,
                      const ORec* R, const OPath* P, int64_t slot) {
  uint64_t rs = stream_for(seed, pid, 0x7E);
  double jx = uni(&rs), jy = uni(&rs);
  const double* cam = S->cam;
  double W = cam[13], H = cam[14], asp = W / H;
  double sx = (2.0 * ((double)px + jx) / W - 1.0) * cam[12] * asp;
  double sy = (1.0 - 2.0 * ((double)py + jy) / H) * cam[12];
  double d[3] = {cam[3] + sx * cam[6] + sy * cam[9], cam[4] + sx * cam[7] + sy * cam[10],
                 cam[5] + sx * cam[8] + sy * cam[11]};
  double inv0 = 1.0 / sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  for (int a = 0; a < 3; ++a) d[a] *= inv0;
  double o[3] = {cam[0], cam[1], cam[2]};
  double est[3] = {0}, beta[3] = {1, 1, 1}, dcam[3] = {0}, camw[3] = {0}, d0n[3] = {0},
         d0p[3] = {0}, efs[3] = {0};
  double epdf = 1.0, rrinv = 1.0;
  int from_cam = 1, allow = 1, n = 0;
  for (;;) {
    int sid;
    double th = nearest(S, o, d, T_EPS, NO_HIT, &sid);
    double pe_dir = pdf_from_hit(S, sid, th, d);
    if (fill && !from_cam) R->pdf_emit_at_phase[off + n - 1] = pe_dir;
    double tev, fw[3];
    int mid;
    int scat = fly(S, o, d, 0.0, th, &rs, &tev, &mid, fw);
    double v[3] = {o[0] + tev * d[0], o[1] + tev * d[1], o[2] + tev * d[2]};
    int vol = 0, cls = -1;
    double k[3] = {0, 0, 0}, g = 0.0, nr[3] = {0, 0, 0};
    if (scat) {
      if (!allow || n >= max_depth) break;
      const double* ss = S->ss[mid];
      double dn = S->mkind[mid] == 0 ? -1.0 : density(S, mid, v) * S->mscale[mid];
      for (int c = 0; c < 3; ++c) k[c] = dn < 0.0 ? ss[c] : ss[c] * dn;
      if (k[0] == 0.0 && k[1] == 0.0 && k[2] == 0.0) break;
      vol = 1;
      g = S->mg[mid];
      cls = mid;
    } else {
      if (sid < 0) break;
      int mat = S->mat[sid];
      for (int a = 0; a < 3; ++a) v[a] = o[a] + th * d[a];
      if (mat == 2) {
        double gn[3];
        normal_at(S, sid, v, gn);
        if (gn[0] * d[0] + gn[1] * d[1] + gn[2] * d[2] < 0.0) {
          const double* ev = S->eval[S->emid[sid]];
          if (from_cam) {
            for (int c = 0; c < 3; ++c) { dcam[c] = fw[c] * ev[c]; est[c] += dcam[c]; }
          } else {
            double den = epdf + pe_dir, cc[3];
            for (int c = 0; c < 3; ++c) { cc[c] = efs[c] * fw[c] * ev[c] / den; est[c] += beta[c] * cc[c]; }
            if (n == 1) for (int c = 0; c < 3; ++c) d0p[c] = cc[c];
            if (fill) {
              int64_t row = off + n - 1;
              for (int c = 0; c < 3; ++c) {
                R->d_phase[row * 3 + c] = fw[c] * ev[c];
                R->i_pt[row * 3 + c] += cc[c];
              }
            }
          }
        }
        break;
      }
      if (mat == 1) break;
      if (!allow || n >= max_depth) break;
      normal_at(S, sid, v, nr);
      if (nr[0] * d[0] + nr[1] * d[1] + nr[2] * d[2] > 0.0)
        for (int a = 0; a < 3; ++a) nr[a] = -nr[a];
      for (int c = 0; c < 3; ++c) k[c] = S->alb[sid][c];
      cls = sid;
    }
    double wc[3];
    for (int c = 0; c < 3; ++c) wc[c] = fw[c] * rrinv;
    for (int c = 0; c < 3; ++c) {
      if (from_cam) { camw[c] = wc[c]; beta[c] = wc[c]; }
      else beta[c] *= (efs[c] / epdf) * wc[c];
    }
    double ax[3] = {d[0], d[1], d[2]};
    ESample es = nee(S, v, &rs);
    double rho_e = vol ? hg(ax[0] * es.w[0] + ax[1] * es.w[1] + ax[2] * es.w[2], g)
                       : pmax(0.0, nr[0] * es.w[0] + nr[1] * es.w[1] + nr[2] * es.w[2]) * (1.0 / PI);
    double cn[3];
    for (int c = 0; c < 3; ++c) {
      double fe = k[c] * rho_e;
      cn[c] = es.delta ? fe * es.rad[c] : fe * es.rad[c] / (es.pdf + rho_e);
      est[c] += beta[c] * cn[c];
    }
    if (n == 0) for (int c = 0; c < 3; ++c) d0n[c] = cn[c];
    double u1 = uni(&rs), u2 = uni(&rs), wp[3], pp;
    if (vol) {
      hg_dir(g, ax, u1, u2, wp);
      pp = hg(ax[0] * wp[0] + ax[1] * wp[1] + ax[2] * wp[2], g);
    } else {
      cos_dir(nr, u1, u2, wp);
      pp = pmax(0.0, nr[0] * wp[0] + nr[1] * wp[1] + nr[2] * wp[2]) * (1.0 / PI);
    }
    double fp[3] = {k[0] * pp, k[1] * pp, k[2] * pp};
    if (fill) {
      int64_t r = off + n;
      for (int a = 0; a < 3; ++a) {
        R->pos[r * 3 + a] = v[a];
        R->omega_out[r * 3 + a] = -ax[a];
        R->normal[r * 3 + a] = nr[a];
        R->coeff[r * 3 + a] = k[a];
        R->phase_dir[r * 3 + a] = wp[a];
        R->emit_dir[r * 3 + a] = es.w[a];
        R->d_emit[r * 3 + a] = es.rad[a];
        R->d_phase[r * 3 + a] = 0.0;
        R->i_pt[r * 3 + a] = cn[a];
        R->w_cont[r * 3 + a] = wc[a];
      }
      R->g[r] = g;
      R->pdf_phase[r] = pp;
      R->pdf_emit_at_phase[r] = 0.0;
      R->pdf_emit[r] = es.pdf;
      R->kind[r] = vol ? 0 : 1;
      R->emit_delta[r] = (uint8_t)es.delta;
      R->class_id[r] = cls;
      R->path_idx[r] = pid;
      R->depth[r] = n;
    }
    ++n;
    if (pp <= 0.0) break;
    rrinv = 1.0;
    allow = 1;
    if (n >= rr_start) {
      double q = (beta[0] * fp[0] / pp + beta[1] * fp[1] / pp + beta[2] * fp[2] / pp) / 3.0;
      if (q > 1.0) q = 1.0;
      if (q < rr_floor) q = rr_floor;
      double u = uni(&rs);
      if (u >= q) allow = 0;
      else rrinv = 1.0 / q;
    }
    for (int c = 0; c < 3; ++c) efs[c] = fp[c];
    epdf = pp;
    from_cam = 0;
    for (int a = 0; a < 3; ++a) {
      o[a] = vol ? v[a] : v[a] + wp[a] * SURF_OFF;
      d[a] = wp[a];
    }
  }
  if (fill && n > 0) {
    double in[3] = {0, 0, 0};
    for (int kk = n - 1; kk >= 0; --kk) {
      int64_t r = off + kk;
      double pp = R->pdf_phase[r];
      for (int c = 0; c < 3; ++c) {
        double dbar = R->i_pt[r * 3 + c];
        R->i_pt[r * 3 + c] = in[c];
        double f = pp > 0.0 ? R->coeff[r * 3 + c] * pp / pp : 0.0;
        in[c] = R->w_cont[r * 3 + c] * (dbar + f * in[c]);
      }
    }
  }
  if (P) {
    for (int c = 0; c < 3; ++c) {
      P->cam_weight[slot * 3 + c] = camw[c];
      P->d_cam[slot * 3 + c] = dcam[c];
      P->direct0[slot * 3 + c] = d0n[c] + d0p[c];
      P->direct0_nee[slot * 3 + c] = d0n[c];
      P->direct0_phase[slot * 3 + c] = d0p[c];
      P->pt_estimate[slot * 3 + c] = est[c];
    }
  }
  return n;
}

/* Paths are handed out in chunks of 256 to a pool of pthreads (results do not
 * depend on the schedule: every path owns its stream and output slots). */
typedef struct {
  const OScene* S;
  int spp, max_depth, rr_start, fill;
  double rr_floor;
  int64_t seed, n;
  int64_t* counts;
  const int64_t* offsets;
  const ORec* R;
  const OPath* P;
  atomic_llong next;
} Job;

static void* worker(void* arg) {
  Job* j = (Job*)arg;
  for (;;) {
    int64_t b = atomic_fetch_add(&j->next, 256);
    if (b >= j->n) return NULL;
    int64_t e = b + 256 < j->n ? b + 256 : j->n;
    for (int64_t p = b; p < e; ++p) {
      int64_t pix = p / j->spp;
      int64_t px = pix % j->S->width, py = pix / j->S->width;
      if (j->fill)
        trace_path(j->S, px, py, p, j->seed, j->max_depth, j->rr_start, j->rr_floor, 1,
                   j->offsets[p], j->R, j->P, p);
      else
        j->counts[p] = trace_path(j->S, px, py, p, j->seed, j->max_depth, j->rr_start,
                                  j->rr_floor, 0, 0, NULL, NULL, 0);
    }
  }
}

static void run(Job* j, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  atomic_init(&j->next, 0);
  for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, worker, j);
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* counts[p] for every path (pass 1) */
void oracle_trace_count(const OScene* S, int spp, int max_depth, int rr_start, double rr_floor,
                        int64_t seed, int64_t* counts, int threads) {
  Job j = {S, spp, max_depth, rr_start, 0, rr_floor, seed, (int64_t)S->width * S->height * spp,
           counts, NULL, NULL, NULL};
  run(&j, threads);
}

/* records at offsets[p] and the path table (pass 2) */
void oracle_trace_fill(const OScene* S, int spp, int max_depth, int rr_start, double rr_floor,
                       int64_t seed, const int64_t* offsets, const ORec* R, const OPath* P,
                       int threads) {
  Job j = {S, spp, max_depth, rr_start, 1, rr_floor, seed, (int64_t)S->width * S->height * spp,
           NULL, offsets, R, P};
  run(&j, threads);
}

int oracle_scene_size(void) { return (int)sizeof(OScene); }

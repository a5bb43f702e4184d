// Volumetric path tracer with record capture (transport/kernels.py).
//
// One thread per camera path, persistent grid-stride over paths.  The
// arithmetic restates trace_one (kernels.py:86-430) and the scenecore njit
// cores it calls in fp64, in the reference's evaluation order, and this
// translation unit is compiled with -fmad=false: with the same splitmix64
// streams (rng.py:19-51) the device reproduces the reference's records up to
// the last-ulp differences of the libm transcendentals.
//
// Record capture is two-pass like the reference (count -> prefix sum ->
// fill, tracer.py:58-70); the backward i_pt sweep (kernels.py:393-408) runs
// over the just-written rows instead of a per-thread stack: the D-bar
// partial sums are staged in the i_pt slot and the f/p factor is recomputed
// from the stored coeff and pdf_phase.
#include <cmath>

#include "common.cuh"

namespace vpg {
namespace {

constexpr double kNoHit = 1e30;
constexpr double kTEps = 1e-7;
constexpr double kSurfOffset = 1e-6;
constexpr double kPi = 3.14159265358979323846;
constexpr double kInvPi = 1.0 / kPi;
constexpr double kInv4Pi = 1.0 / (4.0 * kPi);
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kSaltTrace = 0x7E;
constexpr uint64_t kSaltExtra = 0xED;

enum Mode { kOff = 0, kCount = 1, kFill = 2, kCapture = 3 };

// ---------------------------------------------------------- rng (rng.py)
struct Rng {
  uint64_t s;
  __device__ uint64_t next_u64() {
    s += kGamma;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  __device__ double next() { return double(next_u64() >> 11) * (1.0 / 9007199254740992.0); }
};

__device__ Rng make_stream(int64_t seed, int64_t key, uint64_t salt) {
  Rng r{uint64_t(seed) ^ (uint64_t(key) * 0xD1342543DE82EF95ull)};
  r.s += salt * kGamma;
  const uint64_t z1 = r.next_u64();
  const uint64_t z2 = r.next_u64();
  return Rng{z1 ^ (z2 >> 1)};
}

struct V3 {
  double x, y, z;
};
// reconvergence point: the lanes that are active here wait for each other,
// so a divergent warp runs the code after it together again
__device__ __forceinline__ void reconverge() { __syncwarp(__activemask()); }
// Python's max(a, b) / min(a, b): keep the first unless the second is strictly beyond it
__device__ __forceinline__ double pymax(double a, double b) { return b > a ? b : a; }
__device__ __forceinline__ double pymin(double a, double b) { return b < a ? b : a; }

// ------------------------------------------------------ geometry.py
__device__ void ray_aabb(const V3& o, const V3& d, const double* bd, double& t0, double& t1) {
  t0 = -kNoHit;
  t1 = kNoHit;
  const double oo[3] = {o.x, o.y, o.z}, dd[3] = {d.x, d.y, d.z};
  for (int a = 0; a < 3; ++a) {
    if (dd[a] != 0.0) {
      const double inv = 1.0 / dd[a];
      double lo = (bd[a] - oo[a]) * inv, hi = (bd[3 + a] - oo[a]) * inv;
      if (lo > hi) {
        const double t = lo;
        lo = hi;
        hi = t;
      }
      t0 = pymax(t0, lo);
      t1 = pymin(t1, hi);
    } else if (oo[a] < bd[a] || oo[a] > bd[3 + a]) {
      t0 = 1.0;
      t1 = -1.0;
      return;
    }
  }
}

__device__ V3 quad_normal(double ux, double uy, double uz, double vx, double vy, double vz) {
  const double nx = uy * vz - uz * vy, ny = uz * vx - ux * vz, nz = ux * vy - uy * vx;
  const double inv = 1.0 / sqrt(nx * nx + ny * ny + nz * nz);
  return V3{nx * inv, ny * inv, nz * inv};
}

__device__ double ray_surface(const vpg_scene& sc, int i, const V3& o, const V3& d, double t_min) {
  const double* p = sc.surf_params[i];
  const int type = sc.surf_type[i];
  if (type == 0) {
    const double lx = o.x - p[0], ly = o.y - p[1], lz = o.z - p[2];
    const double b = lx * d.x + ly * d.y + lz * d.z;
    const double c = lx * lx + ly * ly + lz * lz - p[3] * p[3];
    const double disc = b * b - c;
    if (disc < 0.0) return kNoHit;
    const double s = sqrt(disc);
    const double t0 = -b - s;
    if (t0 > t_min) return t0;
    const double t1 = -b + s;
    if (t1 > t_min) return t1;
    return kNoHit;
  }
  if (type == 1) {
    double t0, t1;
    ray_aabb(o, d, p, t0, t1);
    if (t0 > t1) return kNoHit;
    if (t0 > t_min) return t0;
    if (t1 > t_min) return t1;
    return kNoHit;
  }
  const V3 n = quad_normal(p[3], p[4], p[5], p[6], p[7], p[8]);
  const double denom = d.x * n.x + d.y * n.y + d.z * n.z;
  if (fabs(denom) < 1e-12) return kNoHit;
  const double t = ((p[0] - o.x) * n.x + (p[1] - o.y) * n.y + (p[2] - o.z) * n.z) / denom;
  if (t <= t_min) return kNoHit;
  const double hx = o.x + t * d.x - p[0], hy = o.y + t * d.y - p[1], hz = o.z + t * d.z - p[2];
  const double uu = p[3] * p[3] + p[4] * p[4] + p[5] * p[5];
  const double vv = p[6] * p[6] + p[7] * p[7] + p[8] * p[8];
  const double a = (hx * p[3] + hy * p[4] + hz * p[5]) / uu;
  const double b = (hx * p[6] + hy * p[7] + hz * p[8]) / vv;
  if (a < 0.0 || a > 1.0 || b < 0.0 || b > 1.0) return kNoHit;
  return t;
}

// nearest hit, lowest id on ties (geometry.py:145-163)
__device__ double intersect(const vpg_scene& sc, const V3& o, const V3& d, double t_min,
                            double t_max, int& sid) {
  double best = t_max;
  sid = -1;
  for (int i = 0; i < sc.n_surf; ++i) {
    const double t = ray_surface(sc, i, o, d, t_min);
    if (t < best) {
      best = t;
      sid = i;
    }
  }
  return best;
}

__device__ V3 surface_normal_at(const vpg_scene& sc, int i, const V3& x) {
  const double* p = sc.surf_params[i];
  if (sc.surf_type[i] == 0) {
    const double inv = 1.0 / p[3];
    return V3{(x.x - p[0]) * inv, (x.y - p[1]) * inv, (x.z - p[2]) * inv};
  }
  if (sc.surf_type[i] == 1) {
    double best = fabs(x.x - p[0]);
    V3 n{-1.0, 0.0, 0.0};
    double dd = fabs(x.x - p[3]);
    if (dd < best) { best = dd; n = V3{1.0, 0.0, 0.0}; }
    dd = fabs(x.y - p[1]);
    if (dd < best) { best = dd; n = V3{0.0, -1.0, 0.0}; }
    dd = fabs(x.y - p[4]);
    if (dd < best) { best = dd; n = V3{0.0, 1.0, 0.0}; }
    dd = fabs(x.z - p[2]);
    if (dd < best) { best = dd; n = V3{0.0, 0.0, -1.0}; }
    dd = fabs(x.z - p[5]);
    if (dd < best) { n = V3{0.0, 0.0, 1.0}; }
    return n;
  }
  return quad_normal(p[3], p[4], p[5], p[6], p[7], p[8]);
}

// ---------------------------------------------------------- medium.py
// Division by a divisor known ahead: with y = RN(1/b), q = RN(a y),
// r = a - b q (exact, one FMA) and RN(q + r y) is the correctly rounded a / b
// (Markstein's theorem: y within half an ulp of 1/b, q within an ulp of a/b;
// no overflow or underflow, which the tracking quantities never reach).  So
// the tracking loops divide with one DMUL and two DFMA instead of a full
// division sequence each step, bit for bit the same quotients.
struct Divisor {
  double b, y;
  __device__ explicit Divisor(double d) : b(d), y(1.0 / d) {}  // IEEE division: RN(1/d)
  __device__ __forceinline__ double div(double a) const {
    const double q = __dmul_rn(a, y);
    return __fma_rn(__fma_rn(-b, q, a), y, q);
  }
};

__device__ __forceinline__ double grid_density_div(const vpg_scene& sc, int k, const V3& x,
                                                   const Divisor* ext) {
  const double* bd = sc.med_bounds[k];
  const int nx = sc.grid_dims[k][0], ny = sc.grid_dims[k][1], nz = sc.grid_dims[k][2];
  long long ix = (long long)(ext[0].div(x.x - bd[0]) * nx);
  long long iy = (long long)(ext[1].div(x.y - bd[1]) * ny);
  long long iz = (long long)(ext[2].div(x.z - bd[2]) * nz);
  ix = ix < 0 ? 0 : (ix > nx - 1 ? nx - 1 : ix);
  iy = iy < 0 ? 0 : (iy > ny - 1 ? ny - 1 : iy);
  iz = iz < 0 ? 0 : (iz > nz - 1 ? nz - 1 : iz);
  return double(__ldg(sc.grid_data + sc.grid_offset[k] + (iz * ny + iy) * nx + ix));
}

__device__ double grid_density(const vpg_scene& sc, int k, const V3& x) {
  const double* bd = sc.med_bounds[k];
  const int nx = sc.grid_dims[k][0], ny = sc.grid_dims[k][1], nz = sc.grid_dims[k][2];
  long long ix = (long long)((x.x - bd[0]) / (bd[3] - bd[0]) * nx);
  long long iy = (long long)((x.y - bd[1]) / (bd[4] - bd[1]) * ny);
  long long iz = (long long)((x.z - bd[2]) / (bd[5] - bd[2]) * nz);
  ix = ix < 0 ? 0 : (ix > nx - 1 ? nx - 1 : ix);
  iy = iy < 0 ? 0 : (iy > ny - 1 ? ny - 1 : iy);
  iz = iz < 0 ? 0 : (iz > nz - 1 ? nz - 1 : iz);
  return double(__ldg(sc.grid_data + sc.grid_offset[k] + (iz * ny + iy) * nx + ix));
}

struct Flight {
  bool scattered;
  double t;
  double w[3];
};

__device__ Flight flight_one_medium(const vpg_scene& sc, int k, const V3& o, const V3& d,
                                    double a, double b, Rng& rng) {
  const double* st = sc.med_sigma_t[k];
  const double length = b - a;
  Flight f{false, b, {1.0, 1.0, 1.0}};
  if (sc.med_kind[k] == 0) {
    const double sbar = (st[0] + st[1] + st[2]) / 3.0;
    if (sbar <= 0.0) return f;
    const double u = rng.next();
    const double dist = -log1p(-u) / sbar;
    if (dist >= length) {
      for (int c = 0; c < 3; ++c) f.w[c] = exp(-(st[c] - sbar) * length);
      return f;
    }
    for (int c = 0; c < 3; ++c) f.w[c] = exp(-(st[c] - sbar) * dist) / sbar;
    f.scattered = true;
    f.t = a + dist;
    return f;
  }
  const double mu = sc.med_majorant[k];
  if (mu <= 0.0) return f;
  const double scale = sc.med_scale[k];
  const double* bd = sc.med_bounds[k];
  const Divisor dmu(mu), three(3.0);
  const Divisor ext[3] = {Divisor(bd[3] - bd[0]), Divisor(bd[4] - bd[1]), Divisor(bd[5] - bd[2])};
  double t = a;
  while (true) {
    const double u = rng.next();
    t += dmu.div(-log1p(-u));
    if (t >= b) return f;
    const V3 x{o.x + t * d.x, o.y + t * d.y, o.z + t * d.z};
    const double dens = grid_density_div(sc, k, x, ext) * scale;
    const double s0 = st[0] * dens, s1 = st[1] * dens, s2 = st[2] * dens;
    const double sbar = three.div(s0 + s1 + s2);
    const double u2 = rng.next();
    if (u2 * mu < sbar) {
      const double inv = 1.0 / sbar;
      for (int c = 0; c < 3; ++c) f.w[c] *= inv;
      f.scattered = true;
      f.t = t;
      return f;
    }
    // sbar < mu here (u2 < 1), so the divisor is positive
    const Divisor den(mu - sbar);
    f.w[0] *= den.div(mu - s0);
    f.w[1] *= den.div(mu - s1);
    f.w[2] *= den.div(mu - s2);
  }
}

__device__ void transmittance_one_medium(const vpg_scene& sc, int k, const V3& o, const V3& d,
                                         double a, double b, Rng& rng, double* w) {
  const double* st = sc.med_sigma_t[k];
  const double length = b - a;
  w[0] = w[1] = w[2] = 1.0;
  if (length <= 0.0) return;
  if (sc.med_kind[k] == 0) {
    for (int c = 0; c < 3; ++c) w[c] = exp(-st[c] * length);
    return;
  }
  const double mu = sc.med_majorant[k];
  if (mu <= 0.0) return;
  const double scale = sc.med_scale[k];
  const double* bd = sc.med_bounds[k];
  const Divisor dmu(mu);
  const Divisor ext[3] = {Divisor(bd[3] - bd[0]), Divisor(bd[4] - bd[1]), Divisor(bd[5] - bd[2])};
  double t = a;
  while (true) {
    const double u = rng.next();
    t += dmu.div(-log1p(-u));
    if (t >= b) return;
    const V3 x{o.x + t * d.x, o.y + t * d.y, o.z + t * d.z};
    const double dens = grid_density_div(sc, k, x, ext) * scale;
    for (int c = 0; c < 3; ++c) w[c] *= 1.0 - dmu.div(st[c] * dens);
    if (w[0] == 0.0 && w[1] == 0.0 && w[2] == 0.0) {
      w[0] = w[1] = w[2] = 0.0;
      return;
    }
  }
}

struct MediaFlight {
  bool scattered;
  double t;
  int medium;
  double w[3];
};

__device__ MediaFlight media_flight(const vpg_scene& sc, const V3& o, const V3& d, double t_lo,
                                    double t_hi, Rng& rng) {
  MediaFlight mf{false, t_hi, -1, {1.0, 1.0, 1.0}};
  double cur = t_lo;
  for (int it = 0; it < 2 * sc.n_med + 1; ++it) {
    int best_k = -1;
    double best_a = t_hi, best_b = t_hi;
    for (int k = 0; k < sc.n_med; ++k) {
      double t0, t1;
      ray_aabb(o, d, sc.med_bounds[k], t0, t1);
      const double a = pymax(t0, cur), b = pymin(t1, t_hi);
      if (b > a + 1e-12 && a < best_a) {
        best_a = a;
        best_k = k;
        best_b = b;
      }
    }
    if (best_k < 0) return mf;
    const Flight f = flight_one_medium(sc, best_k, o, d, best_a, best_b, rng);
    for (int c = 0; c < 3; ++c) mf.w[c] *= f.w[c];
    if (f.scattered) {
      mf.scattered = true;
      mf.t = f.t;
      mf.medium = best_k;
      return mf;
    }
    cur = best_b + 1e-12;
  }
  return mf;
}

__device__ void media_transmittance(const vpg_scene& sc, const V3& o, const V3& d, double t_lo,
                                    double t_hi, Rng& rng, double* w) {
  w[0] = w[1] = w[2] = 1.0;
  for (int k = 0; k < sc.n_med; ++k) {
    double t0, t1;
    ray_aabb(o, d, sc.med_bounds[k], t0, t1);
    const double a = pymax(t0, t_lo), b = pymin(t1, t_hi);
    if (b > a + 1e-12) {
      double tr[3];
      transmittance_one_medium(sc, k, o, d, a, b, rng, tr);
      for (int c = 0; c < 3; ++c) w[c] *= tr[c];
    }
  }
}

// ----------------------------------------------------------- phase.py
__device__ double hg_pdf(double cs, double g) {
  const double g2 = g * g;
  const double denom = 1.0 + g2 - 2.0 * g * cs;
  return kInv4Pi * (1.0 - g2) / (denom * sqrt(denom));
}

__device__ void make_frame(const V3& n, V3& t, V3& s) {
  double bx = 1.0, by = 0.0, bz = 0.0;
  if (fabs(n.x) > 0.9) {
    bx = 0.0;
    by = 1.0;
  }
  double tx = by * n.z - bz * n.y, ty = bz * n.x - bx * n.z, tz = bx * n.y - by * n.x;
  const double inv = 1.0 / sqrt(tx * tx + ty * ty + tz * tz);
  tx *= inv;
  ty *= inv;
  tz *= inv;
  t = V3{tx, ty, tz};
  s = V3{n.y * tz - n.z * ty, n.z * tx - n.x * tz, n.x * ty - n.y * tx};
}

__device__ V3 orient(const V3& t, const V3& s, const V3& n, double a, double b, double c) {
  const double dx = a * t.x + b * s.x + c * n.x;
  const double dy = a * t.y + b * s.y + c * n.y;
  const double dz = a * t.z + b * s.z + c * n.z;
  const double inv = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
  return V3{dx * inv, dy * inv, dz * inv};
}

__device__ V3 hg_sample_dir(double g, const V3& ax, double u1, double u2) {
  double ct;
  if (fabs(g) < 1e-6) {
    ct = 1.0 - 2.0 * u1;
  } else {
    const double s = (1.0 - g * g) / (1.0 - g + 2.0 * g * u1);
    const double c = (1.0 + g * g - s * s) / (2.0 * g);
    ct = pymin(1.0, pymax(-1.0, c));
  }
  const double st = sqrt(pymax(0.0, 1.0 - ct * ct));
  const double phi = 2.0 * kPi * u2;
  V3 t, s;
  make_frame(ax, t, s);
  const double cp = cos(phi), sp = sin(phi);
  return orient(t, s, ax, st * cp, st * sp, ct);
}

__device__ V3 cosine_sample_dir(const V3& n, double u1, double u2) {
  const double z = sqrt(pymax(1e-12, 1.0 - u2));
  const double r = sqrt(pymax(0.0, u2));
  const double phi = 2.0 * kPi * u1;
  V3 t, s;
  make_frame(n, t, s);
  const double cp = cos(phi), sp = sin(phi);
  return orient(t, s, n, r * cp, r * sp, z);
}

// -------------------------------------------------------- emitters.py
struct EmitterSample {
  V3 w;
  double pdf;
  bool delta;
  double rad[3];
};

// One shadow test (intersect + media transmittance) for every emitter type,
// so the ratio-tracking loop exists once in the kernel: lanes that sampled
// different emitter types reconverge in it (and it is cached once).
__device__ EmitterSample sample_emitter(const vpg_scene& sc, const V3& p, Rng& rng) {
  const int n_em = sc.n_emit;
  const double u = rng.next();
  long long e = (long long)(u * n_em);
  if (e > n_em - 1) e = n_em - 1;
  const double* val = sc.em_value[e];
  const double sel = double(n_em);
  EmitterSample out{V3{0.0, 0.0, 1.0}, 1.0, false, {0.0, 0.0, 0.0}};
  const int type = sc.em_type[e];
  double clear, t_hi, factor;
  if (type == 1) {
    const double* q = sc.em_quad[e];
    const double u1 = rng.next(), u2 = rng.next();
    const double qx = q[0] + u1 * q[3] + u2 * q[6];
    const double qy = q[1] + u1 * q[4] + u2 * q[7];
    const double qz = q[2] + u1 * q[5] + u2 * q[8];
    const double dx = qx - p.x, dy = qy - p.y, dz = qz - p.z;
    const double d2 = dx * dx + dy * dy + dz * dz;
    if (d2 < 1e-16) return out;
    const double dist = sqrt(d2);
    out.w = V3{dx / dist, dy / dist, dz / dist};
    const double* nq = sc.em_normal[e];
    const double cos_q = -(nq[0] * out.w.x + nq[1] * out.w.y + nq[2] * out.w.z);
    out.pdf = d2 / (sc.em_area[e] * pymax(fabs(cos_q), 1e-12) * sel);
    if (cos_q <= 0.0) return out;
    clear = dist - 1e-6 * pymax(1.0, dist);
    t_hi = dist;
    factor = 1.0;  // rad = val * tr
  } else if (type == 0) {
    out.delta = true;
    const double* lp = sc.em_pos[e];
    const double dx = lp[0] - p.x, dy = lp[1] - p.y, dz = lp[2] - p.z;
    const double d2 = dx * dx + dy * dy + dz * dz;
    if (d2 < 1e-16) return out;
    const double dist = sqrt(d2);
    out.w = V3{dx / dist, dy / dist, dz / dist};
    clear = dist - 1e-6 * pymax(1.0, dist);
    t_hi = dist;
    factor = sel / d2;  // rad = val * tr * (sel / d2)
  } else {
    out.delta = true;
    const double* ld = sc.em_pos[e];
    out.w = V3{-ld[0], -ld[1], -ld[2]};
    clear = kNoHit;
    t_hi = kNoHit;
    factor = sel;  // rad = val * tr * sel
  }
  int sid;
  if (intersect(sc, p, out.w, kTEps, clear, sid) < clear) return out;
  double tr[3];
  media_transmittance(sc, p, out.w, 0.0, t_hi, rng, tr);
  // x * 1.0 is exact, so the area light's val * tr rounds as before
  for (int c = 0; c < 3; ++c) out.rad[c] = val[c] * tr[c] * factor;
  return out;
}

__device__ double emitter_dir_pdf_from_hit(const vpg_scene& sc, int sid, double t_hit,
                                           const V3& w) {
  if (sid < 0 || sc.mat_type[sid] != 2) return 0.0;
  const int e = sc.emitter_id[sid];
  if (sc.em_type[e] != 1) return 0.0;
  const double* nq = sc.em_normal[e];
  const double cos_q = fabs(nq[0] * w.x + nq[1] * w.y + nq[2] * w.z);
  if (cos_q < 1e-12) return 0.0;
  return t_hit * t_hit / (sc.em_area[e] * cos_q * sc.n_emit);
}

// Record and path-table stores are streaming (evict-first): the vertex buffer
// is written once per frame and must not push the density grid out of L2.
__device__ __forceinline__ void put3(double* a, int64_t row, double x, double y, double z) {
  __stcs(a + row * 3, x);
  __stcs(a + row * 3 + 1, y);
  __stcs(a + row * 3 + 2, z);
}
template <class T>
__device__ __forceinline__ void put1(T* a, int64_t row, T v) {
  __stcs(a + row, v);
}

struct PathResult {
  int n_rec;
  double est[3];
};

// ------------------------------------------------------- kernels.py
// Capture mode: records go to scratch slots handed out by a warp-aggregated
// counter (paths interleave); a scatter pass later moves them into path
// order and runs the backward i_pt sweep there (k_gather_records), so the tracing
// kernel never walks a path's records back through memory.
struct Capture {
  unsigned long long* counter;
  int64_t capacity;
  double* aos;  // capacity x kScratchDoubles: one record per slot (see RecView)
};

// Record fields.  The capture scratch holds one record per slot, structure
// of arrays would scatter every field store of a path; a slot is
// kScratchDoubles doubles (10 sectors): the doubles at these offsets, then
// path_idx (int64 bits), {class_id, depth} (2 x int32), {kind, emit_delta}.
enum : int {
  kFPos = 0, kFOmega = 3, kFNormal = 6, kFCoeff = 9, kFPhaseDir = 12, kFEmitDir = 15,
  kFDEmit = 18, kFDPhase = 21, kFIpt = 24, kFWcont = 27, kFG = 30, kFPdfPhase = 31,
  kFPdfEap = 32, kFPdfEmit = 33, kFPath = 34, kFClassDepth = 35, kFKind = 36
};

template <int kMode>
struct RecView {
  const vpg_records& soa;
  double* aos;
  // address of field `fld` (component 0) of record `row`
  __device__ __forceinline__ double* f(int fld, int64_t row) const {
    if (kMode == kCapture) return aos + row * VPG_SCRATCH_DOUBLES + fld;
    switch (fld) {
      case kFPos: return soa.pos + row * 3;
      case kFOmega: return soa.omega_out + row * 3;
      case kFNormal: return soa.normal + row * 3;
      case kFCoeff: return soa.coeff + row * 3;
      case kFPhaseDir: return soa.phase_dir + row * 3;
      case kFEmitDir: return soa.emit_dir + row * 3;
      case kFDEmit: return soa.d_emit + row * 3;
      case kFDPhase: return soa.d_phase + row * 3;
      case kFIpt: return soa.i_pt + row * 3;
      case kFWcont: return soa.w_cont + row * 3;
      case kFG: return soa.g + row;
      case kFPdfPhase: return soa.pdf_phase + row;
      case kFPdfEap: return soa.pdf_emit_at_phase + row;
      default: return soa.pdf_emit + row;
    }
  }
  __device__ __forceinline__ void put3(int fld, int64_t row, double x, double y, double z) const {
    double* p = f(fld, row);
    p[0] = x;
    p[1] = y;
    p[2] = z;
  }
  __device__ __forceinline__ void put1(int fld, int64_t row, double v) const { *f(fld, row) = v; }
  __device__ __forceinline__ void put_ints(int64_t row, int64_t path, int32_t cls, int32_t depth,
                                           uint8_t kind, uint8_t delta) const {
    if (kMode == kCapture) {
      double* p = aos + row * VPG_SCRATCH_DOUBLES;
      reinterpret_cast<long long*>(p)[kFPath] = path;
      reinterpret_cast<int2*>(p + kFClassDepth)[0] = make_int2(cls, depth);
      reinterpret_cast<uchar2*>(p + kFKind)[0] = make_uchar2(kind, delta);
    } else {
      soa.path_idx[row] = path;
      soa.class_id[row] = cls;
      soa.depth[row] = depth;
      soa.kind[row] = kind;
      soa.emit_delta[row] = delta;
    }
  }
};

__device__ __forceinline__ int64_t claim_slot(const Capture& cap) {
  const unsigned act = __activemask();
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(act) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(cap.counter, (unsigned long long)__popc(act));
  base = __shfl_sync(act, base, leader);
  return int64_t(base) + __popc(act & ((1u << lane) - 1u));
}

// The per-path state of trace_one (kernels.py:152-391) between bounces, so a
// path can be advanced one bounce at a time: the capture kernel keeps every
// lane busy by starting a new path in a lane whose path ended (the bounce code
// is shared, so lanes at different depths of different paths still execute it
// together).
template <int kMode>
struct PathState {
  Rng rng;
  V3 o, d;
  double est[3], beta[3], dcam[3], camw[3], d0n[3], d0p[3], ext_fs[3];
  double ext_pdf, rr_inv;
  bool from_camera, allow_record;
  int n_rec;
  int64_t path_id, rec_offset, slot;
  // capture: slot of the path's latest record (-1: none yet, or the scratch
  // overflowed); earlier records are reached through Capture::link
  int64_t last_row;
  // row of the path's latest record
  __device__ int64_t last() const { return kMode == kCapture ? last_row : rec_offset + n_rec - 1; }
};

template <int kMode>
__device__ void path_begin(PathState<kMode>& st, const vpg_scene& sc, const vpg_trace_cfg& cfg,
                           int64_t px, int64_t py, int64_t path_id, int64_t rec_offset,
                           int64_t slot) {
  st.path_id = path_id;
  st.rec_offset = rec_offset;
  st.slot = slot;
  st.rng = make_stream(cfg.seed, path_id, kSaltTrace);
  const double jx = st.rng.next();
  const double jy = st.rng.next();
  const double* cam = sc.cam;
  const double width = cam[13], height = cam[14];
  const double aspect = width / height;
  const double sx = (2.0 * (double(px) + jx) / width - 1.0) * cam[12] * aspect;
  const double sy = (1.0 - 2.0 * (double(py) + jy) / height) * cam[12];
  double dx = cam[3] + sx * cam[6] + sy * cam[9];
  double dy = cam[4] + sx * cam[7] + sy * cam[10];
  double dz = cam[5] + sx * cam[8] + sy * cam[11];
  const double inv0 = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
  st.d = V3{dx * inv0, dy * inv0, dz * inv0};
  st.o = V3{cam[0], cam[1], cam[2]};
  for (int c = 0; c < 3; ++c) {
    st.est[c] = 0.0;
    st.beta[c] = 1.0;
    st.dcam[c] = st.camw[c] = st.d0n[c] = st.d0p[c] = st.ext_fs[c] = 0.0;
  }
  st.ext_pdf = 1.0;
  st.rr_inv = 1.0;
  st.from_camera = true;
  st.allow_record = true;
  st.n_rec = 0;
  st.last_row = -1;
}

// One iteration of the bounce loop; false when the path has ended.
template <int kMode>
__device__ bool path_bounce(PathState<kMode>& st, const vpg_scene& sc, const vpg_trace_cfg& cfg,
                            const vpg_records& rec, const Capture& cap) {
  constexpr bool kStore = kMode == kFill || kMode == kCapture;
  Rng& rng = st.rng;
  V3& o = st.o;
  V3& d = st.d;
  double* est = st.est;
  double* beta = st.beta;
  double* dcam = st.dcam;
  double* camw = st.camw;
  double* d0n = st.d0n;
  double* d0p = st.d0p;
  double* ext_fs = st.ext_fs;
  double& ext_pdf = st.ext_pdf;
  double& rr_inv = st.rr_inv;
  bool& from_camera = st.from_camera;
  bool& allow_record = st.allow_record;
  int& n_rec = st.n_rec;
  const int max_depth = cfg.max_depth;
  const int64_t path_id = st.path_id;
  const int64_t rec_offset = st.rec_offset;
  const RecView<kMode> rv{rec, cap.aos};
  int sid;
  const double t_hit = intersect(sc, o, d, kTEps, kNoHit, sid);
  const double pe_at_dir = emitter_dir_pdf_from_hit(sc, sid, t_hit, d);
  if (kStore && !from_camera) {
    const int64_t prow = st.last();
    if (prow >= 0) rv.put1(kFPdfEap, prow, pe_at_dir);
  }
  const MediaFlight mf = media_flight(sc, o, d, 0.0, t_hit, rng);
  V3 v{o.x + mf.t * d.x, o.y + mf.t * d.y, o.z + mf.t * d.z};
  bool volume = false;
  double k[3] = {0, 0, 0};
  double gpar = 0.0;
  V3 nrm{0.0, 0.0, 0.0};
  int class_id = -1;

  if (mf.scattered) {
    if (!allow_record || n_rec >= max_depth) return false;
    const int mid = mf.medium;
    const double* ss = sc.med_sigma_s[mid];
    if (sc.med_kind[mid] == 0) {
      k[0] = ss[0];
      k[1] = ss[1];
      k[2] = ss[2];
    } else {
      const double dens = grid_density(sc, mid, v) * sc.med_scale[mid];
      k[0] = ss[0] * dens;
      k[1] = ss[1] * dens;
      k[2] = ss[2] * dens;
    }
    if (k[0] == 0.0 && k[1] == 0.0 && k[2] == 0.0) return false;  // pure absorption
    volume = true;
    gpar = sc.med_g[mid];
    class_id = mid;
  } else {
    if (sid < 0) return false;
    const int mat = sc.mat_type[sid];
    v = V3{o.x + t_hit * d.x, o.y + t_hit * d.y, o.z + t_hit * d.z};
    if (mat == 2) {
      const V3 gn = surface_normal_at(sc, sid, v);
      if (gn.x * d.x + gn.y * d.y + gn.z * d.z < 0.0) {
        const double* ev = sc.em_value[sc.emitter_id[sid]];
        if (from_camera) {
          for (int c = 0; c < 3; ++c) {
            dcam[c] = mf.w[c] * ev[c];
            est[c] += dcam[c];
          }
        } else {
          const double denom = ext_pdf + pe_at_dir;
          double cc[3];
          for (int c = 0; c < 3; ++c) {
            cc[c] = ext_fs[c] * mf.w[c] * ev[c] / denom;
            est[c] += beta[c] * cc[c];
          }
          if (n_rec == 1)
            for (int c = 0; c < 3; ++c) d0p[c] = cc[c];
          if (kStore) {
            const int64_t row = st.last();
            if (row >= 0) {
              rv.put3(kFDPhase, row, mf.w[0] * ev[0], mf.w[1] * ev[1], mf.w[2] * ev[2]);
              double* ip = rv.f(kFIpt, row);
              for (int c = 0; c < 3; ++c) ip[c] += cc[c];  // staged D-bar
            }
          }
        }
      }
      return false;
    }
    if (mat == 1) return false;  // black absorber
    if (!allow_record || n_rec >= max_depth) return false;
    V3 gn = surface_normal_at(sc, sid, v);
    if (gn.x * d.x + gn.y * d.y + gn.z * d.z > 0.0) gn = V3{-gn.x, -gn.y, -gn.z};
    nrm = gn;
    k[0] = sc.albedo[sid][0];
    k[1] = sc.albedo[sid][1];
    k[2] = sc.albedo[sid][2];
    class_id = sid;
  }

  // ---- record n_rec at v
  double wc[3];
  for (int c = 0; c < 3; ++c) wc[c] = mf.w[c] * rr_inv;
  if (from_camera) {
    for (int c = 0; c < 3; ++c) {
      camw[c] = wc[c];
      beta[c] = wc[c];
    }
  } else {
    for (int c = 0; c < 3; ++c) beta[c] *= (ext_fs[c] / ext_pdf) * wc[c];
  }
  const V3 ax = d;  // arrival direction = phase anchor

  const EmitterSample es = sample_emitter(sc, v, rng);
  double rho_e;
  if (volume) {
    rho_e = hg_pdf(ax.x * es.w.x + ax.y * es.w.y + ax.z * es.w.z, gpar);
  } else {
    rho_e = pymax(0.0, nrm.x * es.w.x + nrm.y * es.w.y + nrm.z * es.w.z) * kInvPi;
  }
  const double p_p_at_e = rho_e;
  double cn[3];
  for (int c = 0; c < 3; ++c) {
    const double fe = k[c] * rho_e;
    cn[c] = es.delta ? fe * es.rad[c] : fe * es.rad[c] / (es.pdf + p_p_at_e);
    est[c] += beta[c] * cn[c];
  }
  if (n_rec == 0)
    for (int c = 0; c < 3; ++c) d0n[c] = cn[c];

  const double u1 = rng.next();
  const double u2 = rng.next();
  V3 wp;
  double pdf_p;
  if (volume) {
    wp = hg_sample_dir(gpar, ax, u1, u2);
    pdf_p = hg_pdf(ax.x * wp.x + ax.y * wp.y + ax.z * wp.z, gpar);
  } else {
    wp = cosine_sample_dir(nrm, u1, u2);
    pdf_p = pymax(0.0, nrm.x * wp.x + nrm.y * wp.y + nrm.z * wp.z) * kInvPi;
  }
  double fp[3];
  for (int c = 0; c < 3; ++c) fp[c] = k[c] * pdf_p;

  int64_t row = -1;
  if (kMode == kFill) row = rec_offset + n_rec;
  // the capture's slot claim below is a warp-synchronous point (active mask,
  // one atomic, a shuffle); the record-free trace gets the same reconvergence
  // here (C4 record-free trace 316 -> 154 ms: without it the divergent lanes
  // of a warp stay apart and run the rest of the bounce one group at a time)
  if (kMode == kOff) reconverge();
  if (kMode == kCapture) {
    const int64_t got = claim_slot(cap);
    row = got < cap.capacity ? got : -1;
    st.last_row = row;
  }
  if (kStore && row >= 0) {
    rv.put3(kFPos, row, v.x, v.y, v.z);
    rv.put3(kFOmega, row, -ax.x, -ax.y, -ax.z);
    rv.put3(kFNormal, row, nrm.x, nrm.y, nrm.z);
    rv.put3(kFCoeff, row, k[0], k[1], k[2]);
    rv.put1(kFG, row, gpar);
    rv.put3(kFPhaseDir, row, wp.x, wp.y, wp.z);
    rv.put1(kFPdfPhase, row, pdf_p);
    rv.put1(kFPdfEap, row, 0.0);
    rv.put3(kFEmitDir, row, es.w.x, es.w.y, es.w.z);
    rv.put1(kFPdfEmit, row, es.pdf);
    rv.put3(kFDEmit, row, es.rad[0], es.rad[1], es.rad[2]);
    rv.put3(kFDPhase, row, 0.0, 0.0, 0.0);
    rv.put3(kFIpt, row, cn[0], cn[1], cn[2]);  // staged D-bar, replaced by the sweep
    rv.put3(kFWcont, row, wc[0], wc[1], wc[2]);
    rv.put_ints(row, path_id, int32_t(class_id), int32_t(n_rec), uint8_t(volume ? 0 : 1),
                uint8_t(es.delta ? 1 : 0));
  }
  ++n_rec;
  if (pdf_p <= 0.0) return false;  // degenerate sample, no continuation

  rr_inv = 1.0;
  allow_record = true;
  if (n_rec >= cfg.rr_start) {
    double q = (beta[0] * fp[0] / pdf_p + beta[1] * fp[1] / pdf_p + beta[2] * fp[2] / pdf_p) / 3.0;
    if (q > 1.0) q = 1.0;
    if (q < cfg.rr_floor) q = cfg.rr_floor;
    const double u = rng.next();
    if (u >= q) allow_record = false;
    else rr_inv = 1.0 / q;
  }
  for (int c = 0; c < 3; ++c) ext_fs[c] = fp[c];
  ext_pdf = pdf_p;
  from_camera = false;
  if (volume) {
    o = v;
  } else {
    o = V3{v.x + wp.x * kSurfOffset, v.y + wp.y * kSurfOffset, v.z + wp.z * kSurfOffset};
  }
  d = wp;
  return true;
}

// One record's step of the backward i_pt sweep (kernels.py:393-408): i_pt
// holds the record's direct term until the sweep replaces it with the
// incoming radiance from the next record; returns this record's outgoing.
__device__ __forceinline__ void sweep_record(double* ip, const double* kcp, const double* wcp,
                                             double pp, double* in) {
  for (int c = 0; c < 3; ++c) {
    const double dbar = ip[c];
    ip[c] = in[c];
    const double kc = kcp[c];
    const double fpp = pp > 0.0 ? kc * pp / pp : 0.0;
    in[c] = wcp[c] * (dbar + fpp * in[c]);
  }
}

// Backward i_pt sweep (fill mode; capture mode sweeps in k_gather_records) and the
// path-table row.
template <int kMode>
__device__ PathResult path_end(PathState<kMode>& st, const vpg_records& rec, const vpg_paths& pth,
                               const Capture& cap) {
  constexpr bool kStore = kMode == kFill || kMode == kCapture;
  const int n_rec = st.n_rec;
  const int64_t slot = st.slot;
  const RecView<kMode> rv{rec, cap.aos};
  const double* est = st.est;
  const double* dcam = st.dcam;
  const double* camw = st.camw;
  const double* d0n = st.d0n;
  const double* d0p = st.d0p;
  if (kMode == kFill && n_rec > 0) {  // backward sweep (kernels.py:393-408)
    double in[3] = {0.0, 0.0, 0.0};
    for (int kk = n_rec - 1; kk >= 0; --kk) {
      const int64_t row = st.rec_offset + kk;
      sweep_record(rv.f(kFIpt, row), rv.f(kFCoeff, row), rv.f(kFWcont, row),
                   *rv.f(kFPdfPhase, row), in);
    }
  }
  if (kMode != kOff) {
    put3(pth.cam_weight, slot, camw[0], camw[1], camw[2]);
    put3(pth.d_cam, slot, dcam[0], dcam[1], dcam[2]);
    put3(pth.direct0, slot, d0n[0] + d0p[0], d0n[1] + d0p[1], d0n[2] + d0p[2]);
    put3(pth.direct0_nee, slot, d0n[0], d0n[1], d0n[2]);
    put3(pth.direct0_phase, slot, d0p[0], d0p[1], d0p[2]);
    put3(pth.pt_estimate, slot, est[0], est[1], est[2]);
    if (kStore) put3(pth.extra_direct, slot, d0n[0] + d0p[0], d0n[1] + d0p[1], d0n[2] + d0p[2]);
  }
  PathResult res{n_rec, {est[0], est[1], est[2]}};
  return res;
}

template <int kMode>
__device__ PathResult trace_one(const vpg_scene& sc, const vpg_trace_cfg& cfg, int64_t px,
                                int64_t py, int64_t path_id, int64_t rec_offset,
                                const vpg_records& rec, const vpg_paths& pth, int64_t slot,
                                const Capture& cap = Capture{nullptr, 0, nullptr}) {
  PathState<kMode> st;
  path_begin(st, sc, cfg, px, py, path_id, rec_offset, slot);
  while (path_bounce(st, sc, cfg, rec, cap)) {
  }
  return path_end(st, rec, pth, cap);
}

// The record-tracing kernels are latency-bound (density reads, fp64
// chains): 64 registers and 32 warps per SM (spilling to L1) beat 128
// registers and 16 warps (C4 capture 190 vs 235 ms, C2 22.3 vs 24.7 ms).  The
// record-free image kernel (a pixel's samples in order per thread) measured
// 10 % slower so, and keeps the compiler's choice.
#ifndef VPG_TRACE_MINB
#define VPG_TRACE_MINB 8
#endif

// count / fill over paths [path_begin, path_begin + path_count)
template <int kMode>
__global__ void __launch_bounds__(128, VPG_TRACE_MINB) k_trace_paths(const vpg_scene sc, const vpg_trace_cfg cfg,
                                                     int64_t* __restrict__ counts,
                                                     const vpg_records rec, const vpg_paths pth) {
  const int64_t spp = cfg.spp;
  const int64_t width = sc.width;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < cfg.path_count;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t path_id = cfg.path_begin + i;
    const int64_t pix = path_id / spp;
    const int64_t off = kMode == kFill ? pth.rec_start[i] : 0;
    const PathResult r = trace_one<kMode>(sc, cfg, pix % width, pix / width, path_id, off, rec,
                                          pth, i);
    if (kMode == kCount) counts[i] = r.n_rec;
  }
}

// Single-pass capture: trace every path once, records into scratch slots.
// A lane whose path ends starts its next path at once (the loop advances
// every lane by one bounce per iteration), so lanes do not idle until the
// longest path of their warp has finished.
#ifndef VPG_TRACE_BLOCK
#define VPG_TRACE_BLOCK 128
#endif
__global__ void __launch_bounds__(VPG_TRACE_BLOCK, VPG_TRACE_MINB * 128 / VPG_TRACE_BLOCK)
k_trace_capture(const vpg_scene sc, const vpg_trace_cfg cfg,
                                                       int64_t* __restrict__ counts,
                                                       const vpg_records scratch,
                                                       const vpg_paths pth, Capture cap) {
  const int64_t spp = cfg.spp;
  const int64_t width = sc.width;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= cfg.path_count) return;
  PathState<kCapture> st;
  {
    const int64_t path_id = cfg.path_begin + i;
    const int64_t pix = path_id / spp;
    path_begin(st, sc, cfg, pix % width, pix / width, path_id, 0, i);
  }
  while (true) {
    if (!path_bounce(st, sc, cfg, scratch, cap)) {
      const PathResult r = path_end(st, scratch, pth, cap);
      counts[i] = r.n_rec;
      i += stride;
      if (i >= cfg.path_count) break;
      const int64_t path_id = cfg.path_begin + i;
      const int64_t pix = path_id / spp;
      path_begin(st, sc, cfg, pix % width, pix / width, path_id, 0, i);
    }
  }
}

// Scratch slot -> its row in path order (rec_start[path] + depth), as an
// inverse map, so the copy below writes the path-ordered records coalesced.
__global__ void k_slot_of_row(const double* __restrict__ aos, int64_t n,
                              const int64_t* __restrict__ rec_start, int64_t path_begin,
                              int32_t* __restrict__ slot_of) {
  for (int64_t sidx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; sidx < n;
       sidx += int64_t(gridDim.x) * blockDim.x) {
    const double* p = aos + sidx * VPG_SCRATCH_DOUBLES;
    const long long pid = reinterpret_cast<const long long*>(p)[kFPath];
    const int depth = reinterpret_cast<const int2*>(p + kFClassDepth)->y;
    slot_of[rec_start[pid - path_begin] + depth] = int32_t(sidx);
  }
}

// Path-ordered SoA records from the slot-major scratch: a warp stages 32
// records (10 full sectors each) in shared memory, runs the backward i_pt
// sweep of every path lying inside those 32 rows there, then writes every
// field of its rows coalesced (lane = row).  A path reaching back before the
// window's first row is listed (its end row) for k_ipt_sweep_listed.
constexpr int kGatherWarps = 4;
#ifndef VPG_GATHER_UNROLL
#define VPG_GATHER_UNROLL 20  // loads in flight per lane (C4 gather: 16.4 ms compiler default, 13.9 at 20)
#endif
constexpr int kGatherUnroll = VPG_GATHER_UNROLL;
constexpr int kSlotStride = VPG_SCRATCH_DOUBLES + 1;  // odd stride: conflict-free row reads
__device__ __forceinline__ long long slot_path(const double* __restrict__ aos,
                                               const int32_t* __restrict__ slot_of, int64_t row) {
  return __double_as_longlong(aos[int64_t(slot_of[row]) * VPG_SCRATCH_DOUBLES + kFPath]);
}
__global__ void __launch_bounds__(kGatherWarps * 32)
k_gather_records(const double* __restrict__ aos, int64_t n, const int32_t* __restrict__ slot_of,
                 const vpg_records dst, int32_t* __restrict__ listed,
                 int32_t* __restrict__ n_listed) {
  __shared__ double buf[kGatherWarps][32 * kSlotStride];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* b = buf[wid];
  const int64_t step = int64_t(gridDim.x) * kGatherWarps * 32;
  for (int64_t base = (int64_t(blockIdx.x) * kGatherWarps + wid) * 32; base < n; base += step) {
    const int cnt = int(n - base < 32 ? n - base : 32);
#pragma unroll kGatherUnroll
    for (int idx = lane; idx < cnt * VPG_SCRATCH_DOUBLES; idx += 32) {
      const int j = idx / VPG_SCRATCH_DOUBLES, w = idx - j * VPG_SCRATCH_DOUBLES;
      b[j * kSlotStride + w] = __ldcs(aos + int64_t(slot_of[base + j]) * VPG_SCRATCH_DOUBLES + w);
    }
    __syncwarp();
    if (lane < cnt) {
      const long long pid = __double_as_longlong(b[lane * kSlotStride + kFPath]);
      const long long next =
          lane + 1 < cnt ? __double_as_longlong(b[(lane + 1) * kSlotStride + kFPath])
                         : (base + cnt < n ? slot_path(aos, slot_of, base + cnt) : -1);
      if (next != pid) {  // the path ends at this row
        int j = lane;
        while (j > 0 && __double_as_longlong(b[(j - 1) * kSlotStride + kFPath]) == pid) --j;
        if (j == 0 && base > 0 && slot_path(aos, slot_of, base - 1) == pid) {
          const int li = atomicAdd(n_listed, 1);
          VPG_CHECK(li <= (n + 31) / 32);  // at most one listed path per window
          listed[li] = int32_t(base + lane);
        } else {
          double in[3] = {0.0, 0.0, 0.0};
          for (int row = lane; row >= j; --row) {
            double* q = b + row * kSlotStride;
            sweep_record(q + kFIpt, q + kFCoeff, q + kFWcont, q[kFPdfPhase], in);
          }
        }
      }
    }
    __syncwarp();
    if (lane < cnt) {
      const int64_t r = base + lane;
      const double* q = b + lane * kSlotStride;
      double* const v3[10] = {dst.pos, dst.omega_out, dst.normal, dst.coeff, dst.phase_dir,
                              dst.emit_dir, dst.d_emit, dst.d_phase, dst.i_pt, dst.w_cont};
      const int off[10] = {kFPos, kFOmega, kFNormal, kFCoeff, kFPhaseDir,
                           kFEmitDir, kFDEmit, kFDPhase, kFIpt, kFWcont};
#pragma unroll
      for (int f = 0; f < 10; ++f)
        for (int c = 0; c < 3; ++c) v3[f][r * 3 + c] = q[off[f] + c];
      dst.g[r] = q[kFG];
      dst.pdf_phase[r] = q[kFPdfPhase];
      dst.pdf_emit_at_phase[r] = q[kFPdfEap];
      dst.pdf_emit[r] = q[kFPdfEmit];
      dst.path_idx[r] = __double_as_longlong(q[kFPath]);
      const long long cd = __double_as_longlong(q[kFClassDepth]);
      dst.class_id[r] = int32_t(cd & 0xFFFFFFFFll);
      dst.depth[r] = int32_t(cd >> 32);
      const long long kd = __double_as_longlong(q[kFKind]);
      dst.kind[r] = uint8_t(kd & 0xFF);
      dst.emit_delta[r] = uint8_t((kd >> 8) & 0xFF);
    }
    __syncwarp();
  }
}

// The backward i_pt sweep of the paths k_gather_records listed (those
// crossing the start of a 32-row window), over the path-ordered records: the
// thread of a listed end row walks the path's rows back (same operations and
// order as path_end's fill-mode sweep, so the same bits).
__global__ void k_ipt_sweep_listed(const vpg_records rec, const int32_t* __restrict__ listed,
                                   const int32_t* __restrict__ n_listed) {
  const int64_t li = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (li >= *n_listed) return;
  const int64_t r = listed[li];
  const int64_t* __restrict__ pidx = rec.path_idx;
  double* __restrict__ ipt = rec.i_pt;
  const double* __restrict__ coeff = rec.coeff;
  const double* __restrict__ wc = rec.w_cont;
  const double* __restrict__ pdf = rec.pdf_phase;
  const int64_t pid = pidx[r];
  int64_t first = r;  // the path's first row
  while (first > 0 && pidx[first - 1] == pid) --first;
  // each row's fields are loaded before the previous row's results are
  // stored (the loads of a row do not wait on the stores of the one after)
  struct Row {
    double ip[3], kc[3], w[3], pp;
  };
  auto load = [&](int64_t row, Row& x) {
    for (int c = 0; c < 3; ++c) {
      x.ip[c] = ipt[row * 3 + c];
      x.kc[c] = coeff[row * 3 + c];
      x.w[c] = wc[row * 3 + c];
    }
    x.pp = pdf[row];
  };
  double in[3] = {0.0, 0.0, 0.0};
  Row cur, nxt;
  load(r, cur);
  for (int64_t row = r; row >= first; --row) {
    if (row > first) load(row - 1, nxt);
    double out[3];
    for (int c = 0; c < 3; ++c) {  // sweep_record's operations
      const double dbar = cur.ip[c];
      out[c] = in[c];
      const double fpp = cur.pp > 0.0 ? cur.kc[c] * cur.pp / cur.pp : 0.0;
      in[c] = cur.w[c] * (dbar + fpp * in[c]);
    }
    for (int c = 0; c < 3; ++c) ipt[row * 3 + c] = out[c];
    cur = nxt;
  }
}

// Record-free PT (render_image_kernel, kernels.py:433-460): paths traced by
// persistent regenerating lanes like the capture (a lane whose path ends
// starts its next one), each path's estimate kept; k_pixel_mean then takes
// every pixel's mean in sample order, the reference's accumulation order,
// so the image is the same bits as one thread per pixel tracing its samples
// in turn (k_trace_image, kept for reference-style single launches).
__global__ void __launch_bounds__(128, VPG_TRACE_MINB)
k_trace_estimates(const vpg_scene sc, const vpg_trace_cfg cfg, int64_t first_path,
                  int64_t n_paths, double* __restrict__ est) {
  const int64_t spp = cfg.spp;
  const int64_t width = sc.width;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n_paths) return;
  const vpg_paths pth{};
  const Capture cap{nullptr, 0, nullptr};
  PathState<kOff> st;
  {
    const int64_t path_id = first_path + i;
    const int64_t pix = path_id / spp;
    path_begin(st, sc, cfg, pix % width, pix / width, path_id, 0, i);
  }
  while (true) {
    if (!path_bounce(st, sc, cfg, vpg_records{}, cap)) {
      const PathResult r = path_end(st, vpg_records{}, pth, cap);
      for (int c = 0; c < 3; ++c) est[i * 3 + c] = r.est[c];
      i += stride;
      if (i >= n_paths) break;
      const int64_t path_id = first_path + i;
      const int64_t pix = path_id / spp;
      path_begin(st, sc, cfg, pix % width, pix / width, path_id, 0, i);
    }
  }
}

__global__ void k_pixel_mean(const double* __restrict__ est, int64_t pix0, int64_t npix, int spp,
                             double* __restrict__ image) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < npix;
       p += int64_t(gridDim.x) * blockDim.x) {
    double acc[3] = {0.0, 0.0, 0.0};
    for (int s = 0; s < spp; ++s)
      for (int c = 0; c < 3; ++c) acc[c] += est[(p * spp + s) * 3 + c];
    for (int c = 0; c < 3; ++c) image[(pix0 + p) * 3 + c] = acc[c] / spp;
  }
}

// record-free image (render_image_kernel): thread per pixel, samples in order
__global__ void __launch_bounds__(128) k_trace_image(const vpg_scene sc, const vpg_trace_cfg cfg,
                                                     double* __restrict__ image) {
  const int64_t npix = int64_t(sc.width) * sc.height;
  const vpg_records rec{};
  const vpg_paths pth{};
  for (int64_t pix = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; pix < npix;
       pix += int64_t(gridDim.x) * blockDim.x) {
    double acc[3] = {0.0, 0.0, 0.0};
    for (int s = 0; s < cfg.spp; ++s) {
      const PathResult r = trace_one<kOff>(sc, cfg, pix % sc.width, pix / sc.width,
                                           pix * cfg.spp + s, 0, rec, pth, 0);
      for (int c = 0; c < 3; ++c) acc[c] += r.est[c];
    }
    for (int c = 0; c < 3; ++c) image[pix * 3 + c] = acc[c] / cfg.spp;
  }
}

// extra_direct_kernel (kernels.py:499-553)
__global__ void __launch_bounds__(128) k_extra_direct(const vpg_scene sc, const vpg_records rec,
                                                      const vpg_paths pth, int64_t path_begin,
                                                      int64_t seed, int n_extra) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < pth.n;
       p += int64_t(gridDim.x) * blockDim.x) {
    if (pth.rec_count[p] == 0) {
      put3(pth.extra_direct, p, 0.0, 0.0, 0.0);
      continue;
    }
    const int64_t r0 = pth.rec_start[p];
    const V3 v{rec.pos[r0 * 3], rec.pos[r0 * 3 + 1], rec.pos[r0 * 3 + 2]};
    const V3 a{-rec.omega_out[r0 * 3], -rec.omega_out[r0 * 3 + 1], -rec.omega_out[r0 * 3 + 2]};
    const V3 n{rec.normal[r0 * 3], rec.normal[r0 * 3 + 1], rec.normal[r0 * 3 + 2]};
    const double kc[3] = {rec.coeff[r0 * 3], rec.coeff[r0 * 3 + 1], rec.coeff[r0 * 3 + 2]};
    const double g = rec.g[r0];
    const bool volume = rec.kind[r0] == 0;
    double acc[3] = {pth.direct0_nee[p * 3], pth.direct0_nee[p * 3 + 1], pth.direct0_nee[p * 3 + 2]};
    Rng rng = make_stream(seed, path_begin + p, kSaltExtra);  // the frame's path index
    for (int i = 0; i < n_extra; ++i) {
      const EmitterSample es = sample_emitter(sc, v, rng);
      const double rho_e = volume ? hg_pdf(a.x * es.w.x + a.y * es.w.y + a.z * es.w.z, g)
                                  : pymax(0.0, n.x * es.w.x + n.y * es.w.y + n.z * es.w.z) * kInvPi;
      for (int c = 0; c < 3; ++c) {
        if (es.delta) acc[c] += kc[c] * rho_e * es.rad[c];
        else acc[c] += kc[c] * rho_e * es.rad[c] / (es.pdf + rho_e);
      }
    }
    const double inv = 1.0 / (1.0 + n_extra);
    put3(pth.extra_direct, p, acc[0] * inv + pth.direct0_phase[p * 3],
         acc[1] * inv + pth.direct0_phase[p * 3 + 1], acc[2] * inv + pth.direct0_phase[p * 3 + 2]);
  }
}

int trace_grid(int64_t work) {
  const int64_t cap = int64_t(sm_count()) * 16;
  int64_t g = (work + 127) / 128;
  return int(g < cap ? g : cap);
}

void check_scene(const vpg_scene& sc) {
  VPG_REQUIRE(sc.n_surf >= 0 && sc.n_surf <= VPG_MAX_SURF, VPG_ELIMIT, "too many surfaces");
  VPG_REQUIRE(sc.n_emit >= 1 && sc.n_emit <= VPG_MAX_EMIT, VPG_ELIMIT, "emitter count out of range");
  VPG_REQUIRE(sc.n_med >= 0 && sc.n_med <= VPG_MAX_MED, VPG_ELIMIT, "too many media");
}

}  // namespace

void trace_image(const vpg_scene& sc, const vpg_trace_cfg& cfg, double* image, cudaStream_t s) {
  check_scene(sc);
  const int64_t npix = int64_t(sc.width) * sc.height, spp = cfg.spp;
  if (npix <= 0 || spp <= 0) {
    VPG_LAUNCH(k_trace_image, trace_grid(npix), 128, 0, s, sc, cfg, image);
    return;
  }
  // pixel ranges whose paths' estimates fit a 2 GB buffer
  const int64_t chunk_pix = std::max<int64_t>(1, (int64_t(2) << 30) / (24 * spp));
  const int64_t max_paths = std::min(npix, chunk_pix) * spp;
  double* est = scratch_of<double>(s, "trace_est", size_t(max_paths) * 3);
  int per_sm = 0;
  VPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &per_sm, reinterpret_cast<const void*>(k_trace_estimates), 128, 0));
  const int64_t wave = int64_t(std::max(per_sm, 1)) * sm_count();
  for (int64_t p0 = 0; p0 < npix; p0 += chunk_pix) {
    const int64_t np = std::min(chunk_pix, npix - p0), n_paths = np * spp;
    const int grid = int(std::min<int64_t>(wave, (n_paths + 127) / 128));
    VPG_LAUNCH(k_trace_estimates, std::max(grid, 1), 128, 0, s, sc, cfg, p0 * spp, n_paths, est);
    VPG_LAUNCH(k_pixel_mean, grid_for(np, 128), 128, 0, s, est, p0, np, int(spp), image);
  }
}

void trace_count(const vpg_scene& sc, const vpg_trace_cfg& cfg, int64_t* counts,
                 const vpg_paths& pth, cudaStream_t s) {
  check_scene(sc);
  VPG_LAUNCH(k_trace_paths<kCount>, trace_grid(cfg.path_count), 128, 0, s, sc, cfg, counts,
             vpg_records{}, pth);
}

void trace_fill(const vpg_scene& sc, const vpg_trace_cfg& cfg, const vpg_records& rec,
                const vpg_paths& pth, cudaStream_t s) {
  check_scene(sc);
  VPG_LAUNCH(k_trace_paths<kFill>, trace_grid(cfg.path_count), 128, 0, s, sc, cfg, nullptr, rec,
             pth);
}

void trace_capture(const vpg_scene& sc, const vpg_trace_cfg& cfg, double* scratch,
                   int64_t capacity, unsigned long long* counter, int64_t* counts,
                   const vpg_paths& pth, cudaStream_t s) {
  check_scene(sc);
  VPG_REQUIRE(capacity >= 0 && capacity < (int64_t(1) << 31), VPG_ELIMIT,
              "capture scratch capacity must be below 2^31 slots");
  VPG_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s));
  // exactly one wave of resident blocks: every lane regenerates paths until
  // the frame is done, so a second wave would only start on the SMs the
  // first frees, late (C4: 168 ms with one wave, 189 with two)
  int per_sm = 0;
  VPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &per_sm, reinterpret_cast<const void*>(k_trace_capture), VPG_TRACE_BLOCK, 0));
  const int64_t wave = int64_t(std::max(per_sm, 1)) * sm_count();
  const int grid =
      int(std::min<int64_t>(wave, (cfg.path_count + VPG_TRACE_BLOCK - 1) / VPG_TRACE_BLOCK));
  VPG_LAUNCH(k_trace_capture, std::max(grid, 1), VPG_TRACE_BLOCK, 0, s, sc, cfg, counts, vpg_records{}, pth,
             Capture{counter, capacity, scratch});
}

void scatter_records(const double* scratch, int64_t n, const int64_t* rec_start,
                     int64_t path_begin, const vpg_records& out, cudaStream_t s) {
  if (n <= 0) return;
  VPG_REQUIRE(n < (int64_t(1) << 31), VPG_ELIMIT, "more than 2^31 records per trace");
  int32_t* slot_of = scratch_of<int32_t>(s, "slot_of_row", size_t(n));
  VPG_LAUNCH(k_slot_of_row, grid_for(n, 256, 1 << 30), 256, 0, s, scratch, n, rec_start, path_begin,
             slot_of);
  const int64_t max_listed = (n + 31) / 32 + 1;
  int32_t* listed = scratch_of<int32_t>(s, "sweep_listed", size_t(max_listed) + 1);
  VPG_CUDA(cudaMemsetAsync(listed + max_listed, 0, sizeof(int32_t), s));
  VPG_LAUNCH(k_gather_records, int((n + 127) / 128 < sm_count() * 8 ? (n + 127) / 128 : sm_count() * 8),
             kGatherWarps * 32, 0, s, scratch, n, slot_of, out, listed, listed + max_listed);
  VPG_LAUNCH(k_ipt_sweep_listed, int((max_listed + 255) / 256), 256, 0, s, out, listed,
             listed + max_listed);
}

// reconstruct_path_estimate (transport/reconstruct.py:52-72): a path's PT
// estimate rebuilt from its records alone, walking them backward with the
// recorded pdfs, weights and raw radiances; the stored i_pt is only
// cross-checked (max |i_pt - recomputed incoming|).  Thread per path, fp64,
// the reference's operation order (this file is built with -fmad=false).
namespace {
__device__ __forceinline__ double rec_strategy(const vpg_records& R, int64_t row, double dx,
                                               double dy, double dz) {
  // phase_pdf_at / the scalar part of scatter_kernel (reconstruct.py:18-36)
  if (R.kind[row] == 0) {
    const double ax = -R.omega_out[row * 3], ay = -R.omega_out[row * 3 + 1],
                 az = -R.omega_out[row * 3 + 2];
    return hg_pdf(ax * dx + ay * dy + az * dz, R.g[row]);
  }
  const double c = R.normal[row * 3] * dx + R.normal[row * 3 + 1] * dy + R.normal[row * 3 + 2] * dz;
  return (c > 0.0 ? c : 0.0) * (1.0 / 3.14159265358979323846);
}

__global__ void k_reconstruct(const vpg_records R, const vpg_paths P, const int64_t* __restrict__ ids,
                              int64_t count, double* __restrict__ est, double* __restrict__ diff) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t p = ids ? ids[i] : i;
    const int64_t start = P.rec_start[p];
    const int32_t cnt = P.rec_count[p];
    double inc[3] = {0.0, 0.0, 0.0};
    double worst = 0.0;
    for (int k = cnt - 1; k >= 0; --k) {
      const int64_t row = start + k;
      for (int c = 0; c < 3; ++c) worst = fmax(worst, fabs(R.i_pt[row * 3 + c] - inc[c]));
      // local_direct_estimate (reconstruct.py:39-49)
      const double ex = R.emit_dir[row * 3], ey = R.emit_dir[row * 3 + 1], ez = R.emit_dir[row * 3 + 2];
      const double px = R.phase_dir[row * 3], py = R.phase_dir[row * 3 + 1], pz = R.phase_dir[row * 3 + 2];
      const double rho_e = rec_strategy(R, row, ex, ey, ez);
      const double rho_p = rec_strategy(R, row, px, py, pz);
      const double den_e = R.emit_delta[row] ? 0.0 : R.pdf_emit[row] + rho_e;
      const double den_p = R.pdf_phase[row] + R.pdf_emit_at_phase[row];
      const double pdf_p = R.pdf_phase[row];
      for (int c = 0; c < 3; ++c) {
        const double co = R.coeff[row * 3 + c];
        const double f_e = co * rho_e, f_p = co * rho_p;
        const double nee = R.emit_delta[row] ? f_e * R.d_emit[row * 3 + c]
                                             : f_e * R.d_emit[row * 3 + c] / den_e;
        const double phase = f_p * R.d_phase[row * 3 + c] / den_p;
        const double dbar = nee + phase;
        const double ratio = pdf_p > 0.0 ? f_p / pdf_p : 0.0;
        inc[c] = R.w_cont[row * 3 + c] * (dbar + ratio * inc[c]);
      }
    }
    for (int c = 0; c < 3; ++c) est[i * 3 + c] = P.d_cam[p * 3 + c] + inc[c];
    diff[i] = worst;
  }
}
}  // namespace

void reconstruct_paths(const vpg_records& rec, const vpg_paths& pth, const int64_t* ids,
                       int64_t count, double* est, double* diff, cudaStream_t s) {
  VPG_REQUIRE(count >= 0, VPG_EINVAL, "negative path count");
  if (!count) return;
  VPG_LAUNCH(k_reconstruct, grid_for(count, 128), 128, 0, s, rec, pth, ids, count, est, diff);
}

void extra_direct(const vpg_scene& sc, const vpg_records& rec, const vpg_paths& pth, int64_t seed,
                  int n_extra, cudaStream_t s, int64_t path_begin) {
  check_scene(sc);
  VPG_REQUIRE(n_extra >= 0, VPG_EINVAL, "n_extra must be >= 0");
  VPG_REQUIRE(path_begin >= 0, VPG_EINVAL, "path_begin must be >= 0");
  VPG_LAUNCH(k_extra_direct, trace_grid(pth.n), 128, 0, s, sc, rec, pth, path_begin, seed, n_extra);
}

}  // namespace vpg

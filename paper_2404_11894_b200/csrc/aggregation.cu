// Build of the aggregation operators (graph.py:94-168) on the device.
//
//   k_pack_members  one coalesced pass over the records (record order) that
//                   transposes what the operators need into a 160-byte
//                   member struct at the record's cluster-major position
//                   (full-sector scattered writes instead of ~17 scattered
//                   field reads per member), plus the continuation parent and
//                   terminal flag of each row.
//   k_aggregate     one CTA per cluster: member geometry staged in shared
//                   memory, every pair's strategy densities evaluated once in
//                   fp64 (HG at g >= 0.9 needs it) and cached as
//                   fp32 for the second pass; p-hat column sums in fp64 with
//                   a fixed reduction order; the s x s kernel block W written
//                   transposed, D-bar and the per-row solve vectors.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <type_traits>
#include <vector>

#include <cub/cub.cuh>

#include "internal.cuh"

namespace vpg {
namespace {

constexpr double kInv4Pi = 1.0 / (4.0 * 3.14159265358979323846);
constexpr double kInvPi = 1.0 / 3.14159265358979323846;
constexpr int kAggThreads = 128;
// HG densities are evaluated all in fp32 for |g| <= kG32 (see hg32)
constexpr float kG32 = 0.95f;
// dynamic shared memory of k_aggregate for the largest supported cluster (2K = 160)
constexpr size_t kAggSmemMax = 226 * 1024;

struct __align__(32) Member {
  double ax, ay, az;  // -omega_out (volume) or the oriented normal (surface)
  double px, py, pz;  // phase_dir
  double ex, ey, ez;  // emit_dir
  double g, pdf_eap, pdf_e;
  float de[3], dp[3];  // d_emit, d_phase
  float coeff[3], wc[3];
  uint32_t flags;  // 1 emit_delta, 2 terminal (no continuation child), 4 surface, 8 |g| > kG32
  int32_t parent;  // cluster-major row of the continuation parent, -1 none / not yet known
  uint32_t pad[2];
};
// five full sectors (i_pt goes straight to i0 from the pack)
static_assert(sizeof(Member) == 160, "Member must stay 5 sectors");

__device__ __forceinline__ double dot3(double ax, double ay, double az, double bx, double by,
                                       double bz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(ax, bx), __dmul_rn(ay, by)), __dmul_rn(az, bz));
}

__device__ __forceinline__ float4 f4(double x, double y, double z) {
  return make_float4(float(x), float(y), float(z), 0.f);
}

// Pack the records list[i] (or off + i when list is null) whose cluster-major
// position is already known (clpos >= 0).
#ifndef VPG_PACK_MINB
#define VPG_PACK_MINB 4  // 64 registers, 32 warps/SM (95 registers left it at 16: 9.2 vs 8.7 ms at C4)
#endif
__global__ void __launch_bounds__(256, VPG_PACK_MINB) k_pack_members(vpg_records rec, const int32_t* __restrict__ clpos,
                               const int32_t* __restrict__ list, int64_t list_n, int64_t off,
                               Member* __restrict__ out, float* __restrict__ term_max,
                               const uint8_t* __restrict__ has_child, float4* __restrict__ i0) {
  const int64_t n = rec.n;
  const int lane = threadIdx.x & 31;
  float tmax[3] = {0.f, 0.f, 0.f};
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < list_n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = list ? int64_t(list[i]) : off + i;
    const int32_t q = clpos[r];
    if (q < 0) continue;
    VPG_CHECK(q < n);
    Member m;
    const bool volume = rec.kind[r] == 0;
    if (volume) {
      m.ax = -rec.omega_out[r * 3];
      m.ay = -rec.omega_out[r * 3 + 1];
      m.az = -rec.omega_out[r * 3 + 2];
    } else {
      m.ax = rec.normal[r * 3];
      m.ay = rec.normal[r * 3 + 1];
      m.az = rec.normal[r * 3 + 2];
    }
    m.px = rec.phase_dir[r * 3];
    m.py = rec.phase_dir[r * 3 + 1];
    m.pz = rec.phase_dir[r * 3 + 2];
    m.ex = rec.emit_dir[r * 3];
    m.ey = rec.emit_dir[r * 3 + 1];
    m.ez = rec.emit_dir[r * 3 + 2];
    m.g = rec.g[r];
    m.pdf_eap = rec.pdf_emit_at_phase[r];
    m.pdf_e = rec.pdf_emit[r];
    for (int c = 0; c < 3; ++c) {
      m.de[c] = float(rec.d_emit[r * 3 + c]);
      m.dp[c] = float(rec.d_phase[r * 3 + c]);
      m.coeff[c] = float(rec.coeff[r * 3 + c]);
      m.wc[c] = float(rec.w_cont[r * 3 + c]);
    }
    // no continuation child (records.py:128-140); shard-local records carry it
    const bool terminal = has_child ? !has_child[r]
                                    : !(r + 1 < n && rec.path_idx[r + 1] == rec.path_idx[r]);
    m.flags = (rec.emit_delta[r] ? 1u : 0u) | (terminal ? 2u : 0u) | (volume ? 0u : 4u) |
              (fabs(m.g) > double(kG32) ? 8u : 0u);
    // continuation parent r-1 (records.py:128-140) when its row is already
    // placed; a parent placed later (a split group) links its children in
    // k_child_links.  Shard-local builds get theirs from k_set_parents.
    m.parent = (!has_child && r > 0 && rec.path_idx[r - 1] == rec.path_idx[r]) ? clpos[r - 1] : -1;
    m.pad[0] = m.pad[1] = 0;
    out[q] = m;
    // I_0 = i_pt (solve.py:72)
    const float ipt[3] = {float(rec.i_pt[r * 3]), float(rec.i_pt[r * 3 + 1]),
                          float(rec.i_pt[r * 3 + 2])};
    i0[q] = make_float4(ipt[0], ipt[1], ipt[2], 0.f);
    if (terminal)
      for (int c = 0; c < 3; ++c) tmax[c] = fmaxf(tmax[c], fabsf(ipt[c]));
  }
  for (int c = 0; c < 3; ++c) {
    float v = tmax[c];
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
    if (lane == 0 && v > 0.f) atomicMax(reinterpret_cast<unsigned int*>(&term_max[c]), __float_as_uint(v));
  }
}

// Children of the records in `list` that were packed before their parent was
// placed (k_pack_members left them -1): row clpos[r+1] propagates into
// clpos[r] when r+1 is on the same path.  Records not placed yet are skipped
// (their own pack links them); a child packed in the same pass already
// carries the same value, so the order against its aggregate is free.
__global__ void k_child_links(vpg_records rec, const int32_t* __restrict__ clpos,
                              const int32_t* __restrict__ list, int64_t list_n,
                              float4* __restrict__ rows) {
  const int64_t n = rec.n;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < list_n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = list[i];
    if (r + 1 >= n || rec.path_idx[r + 1] != rec.path_idx[r]) continue;
    const int32_t q = clpos[r], qc = clpos[r + 1];
    if (q >= 0 && qc >= 0) set_row_parent(rows, qc, q);
  }
}

// Continuation parents, record order: row clpos[r] propagates into clpos[r-1]
// when r-1 is on the same path (records.py:128-140), else nowhere (-1).
__global__ void k_parent_links(vpg_records rec, const int32_t* __restrict__ clpos,
                               float4* __restrict__ rows) {
  const int64_t n = rec.n;
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int32_t par = (r > 0 && rec.path_idx[r - 1] == rec.path_idx[r]) ? clpos[r - 1] : -1;
    set_row_parent(rows, clpos[r], par);
  }
}

// Member l's strategy density toward direction d (graph.py:82-91).  Surface
// members (Lambertian, max(0, n.d)/pi) follow the reference's fp64 rounding
// order exactly, so the zero pattern (and with it the inclusion masks) is
// the reference's.
__device__ __forceinline__ double surface_pdf(const double* __restrict__ geo, int S, int l,
                                              double dx, double dy, double dz) {
  const double cs = dot3(geo[l], geo[S + l], geo[2 * S + l], dx, dy, dz);
  return cs > 0.0 ? __dmul_rn(cs, kInvPi) : 0.0;
}

// Volume members: HG (phase.py:17-21), num / (den * sqrt(den)) with
// den = 1 + g^2 - 2 g cos.  The cosine and den -- where the cancellation at
// g -> 1 lives -- stay fp64; den^-3/2 and the product are fp32 (MUFU rsqrt,
// rel. error ~1e-7 on den's fp32 rounding), which is ~1e-6 on the density,
// far inside the 1e-4 radiance bar, at a quarter of the fp64 issue cost.
// A pdf is never 0 here unless num is (g = +-1), and then in both.
// MUFU reciprocal square root without denormal handling (den is a normal
// number or 0 here)
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float hg_pdf(double ax, double ay, double az, double c1, double c2,
                                        float num, double dx, double dy, double dz) {
  const double cs = fma(az, dz, fma(ay, dy, ax * dx));
  const double den = fma(-c2, cs, c1);
  const float r = rsqrt_ftz(float(den));
  return num * (r * r * r);
}

// Dynamic shared memory for clusters of up to S members:
//   geo   12*S doubles: ax ay az px py pz ex ey ez | HG num c1 c2 (num also
//         as fp32 after them); the fp32 HG clusters (aggregate_v32) keep
//         their packed float4 rows in the same region instead
//   wts    7*S doubles: 1/phat_ind, d_emit/phat_dir_emit (3), d_phase/phat_dir_phase (3)
//          (volume clusters keep them as fp32 in the same region)
//   (the pair densities are not stored: pass 1 sums them into p-hat, pass 2
//   evaluates them again for W and D-bar)
enum AggMode { kSurface = 0, kVol64 = 1, kVol32 = 2 };  // kVol32: aggregate_v32

template <int kMode>
__device__ __forceinline__ void aggregate_cluster(
    const Member* __restrict__ mem, int32_t q0, int s, int64_t wb, int64_t n, int S,
    double* __restrict__ geo, double* __restrict__ wts, float* __restrict__ wt, double* __restrict__ phat, float4* __restrict__ dbar_o,
    float4* __restrict__ coeff_o, float4* __restrict__ rows_o) {
  constexpr bool kVol = kMode != kSurface;
  using acc_t = typename std::conditional<kVol, float, double>::type;
  const int tid = threadIdx.x;
  const float* numf = reinterpret_cast<const float*>(geo + 12 * S);  // S floats after geo
  float* wtsf = reinterpret_cast<float*>(wts);
  const double ks = double(s);

  // pass 1: columns j, P threads per column (P = 4 for s <= 32, else 2) each
  // summing a contiguous slice of l; the slices combine in a fixed order
  // (((p0 + p1) + (p2 + p3))), so p-hat is deterministic.  The loop trip
  // count is uniform so every lane reaches the shuffles.
  const int P = s <= 32 ? 4 : 2;
  const int slice = (s + P - 1) / P;
  for (int base = 0; base < P * s; base += blockDim.x) {
    const int t = base + tid;
    const bool active = t < P * s;
    const int j = t / P, h = t % P;
    acc_t sp = 0, se = 0;
    if (active) {
      const int l0 = h * slice, l1 = min(s, l0 + slice);
      {
        const double dpx = geo[3 * S + j], dpy = geo[4 * S + j], dpz = geo[5 * S + j];
        const double dex = geo[6 * S + j], dey = geo[7 * S + j], dez = geo[8 * S + j];
        for (int l = l0; l < l1; ++l) {
          if constexpr (kMode == kVol64) {
            const double ax = geo[l], ay = geo[S + l], az = geo[2 * S + l];
            const double c1 = geo[10 * S + l], c2 = geo[11 * S + l];
            const float a = hg_pdf(ax, ay, az, c1, c2, numf[l], dpx, dpy, dpz);
            const float b = hg_pdf(ax, ay, az, c1, c2, numf[l], dex, dey, dez);
            sp += a;
            se += b;
          } else {
            const double a = surface_pdf(geo, S, l, dpx, dpy, dpz);
            const double b = surface_pdf(geo, S, l, dex, dey, dez);
            sp = __dadd_rn(sp, a);
            se = __dadd_rn(se, b);
          }
        }
      }
    }
    sp += __shfl_xor_sync(0xFFFFFFFFu, sp, 1);
    se += __shfl_xor_sync(0xFFFFFFFFu, se, 1);
    if (P == 4) {
      sp += __shfl_xor_sync(0xFFFFFFFFu, sp, 2);
      se += __shfl_xor_sync(0xFFFFFFFFu, se, 2);
    }
    if (active && h == 0) {
      const Member& mb = mem[q0 + j];
      const double p_ind = double(sp);
      const double p_dp = __dadd_rn(p_ind, __dmul_rn(ks, mb.pdf_eap));
      const double p_de = (mb.flags & 1u) ? ks : __dadd_rn(double(se), __dmul_rn(ks, mb.pdf_e));
      const int64_t q = q0 + j;
      phat[q] = p_ind;
      phat[n + q] = p_dp;
      phat[2 * n + q] = p_de;
      const bool inc_p = isfinite(p_ind) && p_ind > 0.0;
      const bool inc_e = isfinite(p_de) && p_de > 0.0;
      const bool ok_dp = inc_p && isfinite(p_dp) && p_dp > 0.0;
      const double ie = inc_e ? __ddiv_rn(1.0, p_de) : 0.0;
      const double ip = ok_dp ? __ddiv_rn(1.0, p_dp) : 0.0;
      const double iw = inc_p ? __ddiv_rn(1.0, p_ind) : 0.0;
      if constexpr (kVol) {
        wtsf[j] = float(iw);
        wtsf[S + j] = float(double(mb.de[0]) * ie);
        wtsf[2 * S + j] = float(double(mb.de[1]) * ie);
        wtsf[3 * S + j] = float(double(mb.de[2]) * ie);
        wtsf[4 * S + j] = float(double(mb.dp[0]) * ip);
        wtsf[5 * S + j] = float(double(mb.dp[1]) * ip);
        wtsf[6 * S + j] = float(double(mb.dp[2]) * ip);
      } else {
        wts[j] = iw;
        wts[S + j] = double(mb.de[0]) * ie;
        wts[2 * S + j] = double(mb.de[1]) * ie;
        wts[3 * S + j] = double(mb.de[2]) * ie;
        wts[4 * S + j] = double(mb.dp[0]) * ip;
        wts[5 * S + j] = double(mb.dp[1]) * ip;
        wts[6 * S + j] = double(mb.dp[2]) * ip;
      }
    }
  }
  __syncthreads();

  // pass 2: rows: the kernel block (transposed, wt[wb + j*s + r] = W[r, j]),
  // D-bar and the solve vectors, P2 threads per row each covering a slice
  // of the columns, the D-bar sums combined in a fixed order
  const int P2 = s <= 32 ? 4 : 2;
  const int slice2 = (s + P2 - 1) / P2;
  for (int base = 0; base < P2 * s; base += blockDim.x) {
    const int t = base + tid;
    const bool active = t < P2 * s;
    const int r = t / P2, h = t % P2;
    acc_t dx = 0, dy = 0, dz = 0;
    if (active) {
      const int j0 = h * slice2, j1 = min(s, j0 + slice2);
      // both densities are recomputed rather than kept in shared memory: no
      // pair storage, 16 CTAs per SM instead of 8
      if constexpr (kMode == kVol64) {
        const double ax = geo[r], ay = geo[S + r], az = geo[2 * S + r];
        const double c1 = geo[10 * S + r], c2 = geo[11 * S + r];
        const float num = numf[r];
        for (int j = j0; j < j1; ++j) {
          const float a = hg_pdf(ax, ay, az, c1, c2, num, geo[3 * S + j], geo[4 * S + j],
                                 geo[5 * S + j]);
          wt[wb + j * s + r] = a * wtsf[j];
          const float b = hg_pdf(ax, ay, az, c1, c2, num, geo[6 * S + j], geo[7 * S + j],
                                 geo[8 * S + j]);
          dx += b * wtsf[S + j] + a * wtsf[4 * S + j];
          dy += b * wtsf[2 * S + j] + a * wtsf[5 * S + j];
          dz += b * wtsf[3 * S + j] + a * wtsf[6 * S + j];
        }
      } else {
        for (int j = j0; j < j1; ++j) {
          const double a = surface_pdf(geo, S, r, geo[3 * S + j], geo[4 * S + j], geo[5 * S + j]);
          wt[wb + j * s + r] = float(a * wts[j]);
          const double b = surface_pdf(geo, S, r, geo[6 * S + j], geo[7 * S + j], geo[8 * S + j]);
          dx += b * wts[S + j] + a * wts[4 * S + j];
          dy += b * wts[2 * S + j] + a * wts[5 * S + j];
          dz += b * wts[3 * S + j] + a * wts[6 * S + j];
        }
      }
    }
    dx += __shfl_xor_sync(0xFFFFFFFFu, dx, 1);
    dy += __shfl_xor_sync(0xFFFFFFFFu, dy, 1);
    dz += __shfl_xor_sync(0xFFFFFFFFu, dz, 1);
    if (P2 == 4) {
      dx += __shfl_xor_sync(0xFFFFFFFFu, dx, 2);
      dy += __shfl_xor_sync(0xFFFFFFFFu, dy, 2);
      dz += __shfl_xor_sync(0xFFFFFFFFu, dz, 2);
    }
    if (active && h == 0) {
      const Member& mb = mem[q0 + r];
      const double kx = mb.coeff[0], ky = mb.coeff[1], kz = mb.coeff[2];
      const double bx = kx * double(dx), by = ky * double(dy), bz = kz * double(dz);
      const double wx = mb.wc[0], wy = mb.wc[1], wz = mb.wc[2];
      const int64_t q = q0 + r;
      dbar_o[q] = f4(bx, by, bz);
      coeff_o[q] = f4(kx, ky, kz);
      // row layout (graph.cuh): {a, link}, {b, 1/phat_ind}, {HG anchor, g},
      // {phase direction, 1 - |d|^2}; link = (parent + 1) * 2 + terminal
      // (terminal: no continuation child writes the row, the solve carries
      // its I over from iteration to iteration)
      rows_o[4 * q] = make_float4(float(wx * kx), float(wy * ky), float(wz * kz),
                                  __int_as_float(row_link(mb.parent, mb.flags & 2u)));
      // (the fp32 HG clusters are aggregated by aggregate_v32; these rows'
      // anchor / direction slots are not read by the solve)
      const float iw = kVol ? wtsf[r] : float(wts[r]);
      const float ax = float(geo[r]), ay = float(geo[S + r]), az = float(geo[2 * S + r]);
      const float g = float(mb.g);
      const float dx3 = float(geo[3 * S + r]), dy3 = float(geo[4 * S + r]),
                  dz3 = float(geo[5 * S + r]), cd = 0.f;
      rows_o[4 * q + 1] = make_float4(float(wx * bx), float(wy * by), float(wz * bz), iw);
      rows_o[4 * q + 2] = make_float4(ax, ay, az, g);
      rows_o[4 * q + 3] = make_float4(dx3, dy3, dz3, cd);
    }
  }
}

// fp32 HG clusters (volume members, |g| <= kG32).  Every operand is fp32:
// den = 1 + g^2 - 2g cos is evaluated as |d - g a|^2 + (1 - |d|^2) (+ g^2
// (1 - |a|^2), ~1e-16 for the unit anchors and left out), an identity in
// which nothing cancels: for |g| <= 0.95 the components of d - g a are
// >= ~0.05 in the forward peak, so the fp32 rounding of the inputs costs
// < 1e-5 relative on the density (measured ~1e-6), inside the 1e-4 radiance
// bar; larger |g| keeps the fp64 cosine and denominator (hg_pdf above).  The
// member data is packed as float4 rows so every pair costs two shared-memory
// loads per density:
//   A4[l] = {anchor, g}, NM[l] = num(g), P4[j] = {phase_dir, 1 - |d|^2},
//   E4[j] = {emit_dir, 1 - |e|^2}, WE4[j] = {d_emit / phat_dir_emit, 1/phat_ind},
//   WP4[j] = {d_phase / phat_dir_phase, 0}.
// hg32 is the same arithmetic as the solve's recomputed W (operators.cu
// w_recomputed), so both see the same W bit for bit.
__device__ __forceinline__ float hg32(const float4 a, float num, const float4 d) {
  const float ux = fmaf(-a.w, a.x, d.x), uy = fmaf(-a.w, a.y, d.y), uz = fmaf(-a.w, a.z, d.z);
  const float r = rsqrt_ftz(fmaf(ux, ux, fmaf(uy, uy, fmaf(uz, uz, d.w))));
  return num * (r * r * r);
}

__device__ __forceinline__ void aggregate_v32(
    const Member* __restrict__ mem, int32_t q0, int s, int64_t n, const float4* __restrict__ A4,
    const float* __restrict__ NM, const float4* __restrict__ P4, const float4* __restrict__ E4,
    float4* __restrict__ WE4, float4* __restrict__ WP4, double* __restrict__ phat,
    float4* __restrict__ dbar_o, float4* __restrict__ coeff_o, float4* __restrict__ rows_o) {
  const int tid = threadIdx.x;
  const double ks = double(s);
  // column sums, then row sums, handed from the passes to their per-member
  // epilogues (free space after WP4 in the weights region: 16 S bytes)
  float2* SS = reinterpret_cast<float2*>(WP4 + s);
  float4* DS = reinterpret_cast<float4*>(WP4 + s);
  // pass 1: columns (P threads each, fixed combination order), p-hat, weights
  const int P = s <= 32 ? 4 : 2;
  for (int base = 0; base < P * s; base += blockDim.x) {
    const int t = base + tid;
    const bool active = t < P * s;
    const int j = t / P, h = t % P;
    float sp = 0.f, se = 0.f;
    if (active) {
      // thread h takes every P-th member (strided, not a contiguous slice:
      // the P threads of a column then read consecutive rows of A4 -- no
      // shared-memory bank conflicts); the P partial sums combine in a fixed
      // order, so p-hat stays deterministic
      const float4 pj = P4[j], ej = E4[j];
      for (int l = h; l < s; l += P) {
        const float4 a = A4[l];
        const float num = NM[l];
        sp += hg32(a, num, pj);
        se += hg32(a, num, ej);
      }
    }
    sp += __shfl_xor_sync(0xFFFFFFFFu, sp, 1);
    se += __shfl_xor_sync(0xFFFFFFFFu, se, 1);
    if (P == 4) {
      sp += __shfl_xor_sync(0xFFFFFFFFu, sp, 2);
      se += __shfl_xor_sync(0xFFFFFFFFu, se, 2);
    }
    if (active && h == 0) SS[j] = make_float2(sp, se);
  }
  __syncthreads();
  // the per-member marginals and weights, one member per thread (fp64
  // divisions: with P lanes per column most of a warp would idle here)
  for (int j = tid; j < s; j += blockDim.x) {
    {
      const float sp = SS[j].x, se = SS[j].y;
      const Member& mb = mem[q0 + j];
      const double p_ind = double(sp);
      const double p_dp = __dadd_rn(p_ind, __dmul_rn(ks, mb.pdf_eap));
      const double p_de = (mb.flags & 1u) ? ks : __dadd_rn(double(se), __dmul_rn(ks, mb.pdf_e));
      const int64_t q = q0 + j;
      phat[q] = p_ind;
      phat[n + q] = p_dp;
      phat[2 * n + q] = p_de;
      const bool inc_p = isfinite(p_ind) && p_ind > 0.0;
      const bool inc_e = isfinite(p_de) && p_de > 0.0;
      const bool ok_dp = inc_p && isfinite(p_dp) && p_dp > 0.0;
      const double ie = inc_e ? __ddiv_rn(1.0, p_de) : 0.0;
      const double ip = ok_dp ? __ddiv_rn(1.0, p_dp) : 0.0;
      const double iw = inc_p ? __ddiv_rn(1.0, p_ind) : 0.0;
      WE4[j] = make_float4(float(double(mb.de[0]) * ie), float(double(mb.de[1]) * ie),
                           float(double(mb.de[2]) * ie), float(iw));
      WP4[j] = make_float4(float(double(mb.dp[0]) * ip), float(double(mb.dp[1]) * ip),
                           float(double(mb.dp[2]) * ip), 0.f);
    }
  }
  __syncthreads();
  // pass 2: rows -- D-bar and the solve's row data (no W block: recomputed)
  const int P2 = s <= 32 ? 4 : 2;
  for (int base = 0; base < P2 * s; base += blockDim.x) {
    const int t = base + tid;
    const bool active = t < P2 * s;
    const int r = t / P2, h = t % P2;
    float dx = 0.f, dy = 0.f, dz = 0.f;
    if (active) {
      const float4 a = A4[r];
      const float num = NM[r];
      for (int j = h; j < s; j += P2) {  // strided columns (see pass 1)
        const float pa = hg32(a, num, P4[j]);
        const float pb = hg32(a, num, E4[j]);
        const float4 we = WE4[j], wp = WP4[j];
        dx += pb * we.x + pa * wp.x;
        dy += pb * we.y + pa * wp.y;
        dz += pb * we.z + pa * wp.z;
      }
    }
    dx += __shfl_xor_sync(0xFFFFFFFFu, dx, 1);
    dy += __shfl_xor_sync(0xFFFFFFFFu, dy, 1);
    dz += __shfl_xor_sync(0xFFFFFFFFu, dz, 1);
    if (P2 == 4) {
      dx += __shfl_xor_sync(0xFFFFFFFFu, dx, 2);
      dy += __shfl_xor_sync(0xFFFFFFFFu, dy, 2);
      dz += __shfl_xor_sync(0xFFFFFFFFu, dz, 2);
    }
    if (active && h == 0) DS[r] = make_float4(dx, dy, dz, 0.f);
  }
  __syncthreads();
  // D-bar and the row data, one member per thread
  for (int r = tid; r < s; r += blockDim.x) {
    {
      const float dx = DS[r].x, dy = DS[r].y, dz = DS[r].z;
      const Member& mb = mem[q0 + r];
      const double kx = mb.coeff[0], ky = mb.coeff[1], kz = mb.coeff[2];
      const double bx = kx * double(dx), by = ky * double(dy), bz = kz * double(dz);
      const double wx = mb.wc[0], wy = mb.wc[1], wz = mb.wc[2];
      const int64_t q = q0 + r;
      dbar_o[q] = f4(bx, by, bz);
      coeff_o[q] = f4(kx, ky, kz);
      rows_o[4 * q] = make_float4(float(wx * kx), float(wy * ky), float(wz * kz),
                                  __int_as_float(row_link(mb.parent, mb.flags & 2u)));
      rows_o[4 * q + 1] = make_float4(float(wx * bx), float(wy * by), float(wz * bz), WE4[r].w);
      rows_o[4 * q + 2] = A4[r];
      rows_o[4 * q + 3] = P4[r];
    }
  }
}

__global__ void __launch_bounds__(kAggThreads, 10)
k_aggregate(const Member* __restrict__ mem, const int32_t* __restrict__ cl_off,
            const int32_t* __restrict__ cl_size, const int64_t* __restrict__ w_off,
            const int64_t* __restrict__ range, int64_t n, int S,
            float* __restrict__ wt, double* __restrict__ phat, float4* __restrict__ dbar_o,
            float4* __restrict__ coeff_o, float4* __restrict__ rows_o,
            uint8_t* __restrict__ cl_mode) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* geo = reinterpret_cast<double*>(smem);
  float* numf = reinterpret_cast<float*>(geo + 12 * S);
  double* wts = geo + 12 * S + (S + 1) / 2;
  // fp32 HG clusters: packed float4 member data in the same space
  float4* A4 = reinterpret_cast<float4*>(geo);
  float4* P4 = A4 + S;
  float4* E4 = P4 + S;
  float* NM = reinterpret_cast<float*>(E4 + S);  // 52 S bytes <= the 96 S of geo
  float4* WE4 = reinterpret_cast<float4*>((reinterpret_cast<uintptr_t>(wts) + 15) & ~uintptr_t(15));
  float4* WP4 = WE4 + S;  // 32 S + 15 bytes <= the 56 S of wts
  const int tid = threadIdx.x;

  const int64_t k_end = range[1];
  for (int64_t k = range[0] + blockIdx.x; k < k_end; k += gridDim.x) {
    const int32_t q0 = cl_off[k];
    const int s = cl_size[k];
    const int64_t wb = w_off[k];
    {
      // pull the next cluster's members towards L2 while this one computes
      const int64_t kn = k + gridDim.x;
      if (kn < k_end) {
        const int32_t qn = cl_off[kn], sn = cl_size[kn];
        const char* base = reinterpret_cast<const char*>(mem + qn);
        const int lines = (sn * int(sizeof(Member)) + 127) / 128;
        for (int i = tid; i < lines; i += blockDim.x)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(base + 128 * i));
      }
    }
    // the cluster's mode: Lambertian, HG with fp64 denominators (some
    // |g| > kG32), or HG all in fp32 -- every warp reduces the member flags
    // itself, so no block barrier is needed
    uint32_t fl = 0;
    for (int l = tid & 31; l < s; l += 32) fl |= mem[q0 + l].flags;
    const bool surface = __any_sync(0xFFFFFFFFu, fl & 4u);
    const bool need64 = __any_sync(0xFFFFFFFFu, fl & 8u);
    const int mode = surface ? kSurface : (need64 ? kVol64 : kVol32);
    // 1: W block stored (Lambertian / |g| > kG32), 0: recomputed by the solve
    if (tid == 0) cl_mode[k] = mode == kVol32 ? 0 : 1;
    for (int l = tid; l < s; l += blockDim.x) {
      const Member& mb = mem[q0 + l];
      const double g = mb.g;
      const double g2 = __dmul_rn(g, g);
      const double num = __dmul_rn(kInv4Pi, __dsub_rn(1.0, g2));
      if (mode == kVol32) {
        // g^2 (1 - |a|^2) is ~1e-16 for the unit anchors: left out here and in
        // the solve's recomputed blocks, so both evaluate the same W; num is
        // the solve's own fp32 normalisation
        const double np = fma(mb.px, mb.px, fma(mb.py, mb.py, mb.pz * mb.pz));
        const double ne = fma(mb.ex, mb.ex, fma(mb.ey, mb.ey, mb.ez * mb.ez));
        A4[l] = make_float4(float(mb.ax), float(mb.ay), float(mb.az), float(g));
        P4[l] = make_float4(float(mb.px), float(mb.py), float(mb.pz), float(1.0 - np));
        E4[l] = make_float4(float(mb.ex), float(mb.ey), float(mb.ez), float(1.0 - ne));
        NM[l] = hg_num_f32(float(g));
      } else {
        geo[l] = mb.ax;
        geo[S + l] = mb.ay;
        geo[2 * S + l] = mb.az;
        geo[3 * S + l] = mb.px;
        geo[4 * S + l] = mb.py;
        geo[5 * S + l] = mb.pz;
        geo[6 * S + l] = mb.ex;
        geo[7 * S + l] = mb.ey;
        geo[8 * S + l] = mb.ez;
        geo[9 * S + l] = num;
        numf[l] = float(num);
        geo[10 * S + l] = __dadd_rn(1.0, g2);
        geo[11 * S + l] = __dmul_rn(2.0, g);
      }
    }
    __syncthreads();
    if (mode == kVol32)
      aggregate_v32(mem, q0, s, n, A4, NM, P4, E4, WE4, WP4, phat, dbar_o, coeff_o, rows_o);
    else if (mode == kVol64)
      aggregate_cluster<kVol64>(mem, q0, s, wb, n, S, geo, wts, wt, phat, dbar_o, coeff_o,
                                rows_o);
    else
      aggregate_cluster<kSurface>(mem, q0, s, wb, n, S, geo, wts, wt, phat, dbar_o, coeff_o,
                                  rows_o);
    __syncthreads();
  }
}

// Shard-local parents: given directly (a halo slot n + h for a parent on
// another shard, -1 for none).
__global__ void k_set_parents(const int32_t* __restrict__ parent, int64_t n,
                              float4* __restrict__ rows) {
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < n;
       q += int64_t(gridDim.x) * blockDim.x)
    set_row_parent(rows, q, parent[q]);
}

// I_0 of the halo slots: the remote parent's i_pt (solve.py:72, I_0 = i_pt).
__global__ void k_halo_i0(const double* __restrict__ ipt, int64_t n_halo, float4* __restrict__ i0) {
  for (int64_t h = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; h < n_halo;
       h += int64_t(gridDim.x) * blockDim.x)
    i0[h] = make_float4(float(ipt[3 * h]), float(ipt[3 * h + 1]), float(ipt[3 * h + 2]), 0.f);
}

__global__ void k_iota32(int32_t* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = int32_t(i);
}

__global__ void k_cluster_of_rows(const int32_t* __restrict__ cl_off, int64_t m,
                                  int32_t* __restrict__ cluster_id) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < m;
       k += int64_t(gridDim.x) * blockDim.x)
    for (int32_t q = cl_off[k]; q < cl_off[k + 1]; ++q) cluster_id[q] = int32_t(k);
}

// Solve chunks (see graph.cuh): cost prefix and the first cluster of each chunk.
// cost[k]: staged floats of cluster k (its W block only when stored, the
// row data, I and the previous W*I); wcost[k]: its staged W floats.
__global__ void k_chunk_cost(const int32_t* __restrict__ cl_off, const uint8_t* __restrict__ cl_mode,
                             int64_t m, int64_t* __restrict__ cost, int64_t* __restrict__ wcost) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k <= m;
       k += int64_t(gridDim.x) * blockDim.x) {
    if (k == m) { cost[k] = 0; wcost[k] = 0; continue; }
    const int64_t s = cl_off[k + 1] - cl_off[k];
    const int64_t w = cl_mode[k] ? ((s * s + 3) & ~int64_t(3)) : 0;
    cost[k] = w + kRowFloats * s + 4;
    wcost[k] = w;
  }
}

__global__ void k_chunk_first(const int64_t* __restrict__ cst, int64_t m, int64_t cap,
                              int64_t chunk_floats, int32_t* __restrict__ first,
                              int64_t* __restrict__ n_chunks_out) {
  const int64_t n_chunks = (cst[m] + chunk_floats - 1) / chunk_floats;  // <= cap
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_chunks_out = n_chunks;
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c <= n_chunks && c <= cap;
       c += int64_t(gridDim.x) * blockDim.x) {
    if (c == n_chunks) { first[c] = int32_t(m); continue; }
    const int64_t target = c * chunk_floats;
    int64_t lo = 0, hi = m;  // first k with cst[k] >= target
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (cst[mid] < target) lo = mid + 1; else hi = mid;
    }
    first[c] = int32_t(lo);
  }
}

// Chunk descriptors (one 32-byte load per chunk for the solve's producer) and
// the per-cluster table staged with each chunk.  Cluster k is in chunk
// floor(cst[k] / chunk_floats) (chunk_first[c] = first k with cst[k] >= c F).
// Chunk descriptors: {k0, nk, q0, R} and {staged W floats, 0, 0, 0}.
__global__ void k_chunk_desc(const int32_t* __restrict__ first, const int64_t* __restrict__ n_chunks_p,
                             const int32_t* __restrict__ cl_off, const int64_t* __restrict__ wcs,
                             int4* __restrict__ desc) {
  const int64_t n_chunks = *n_chunks_p;
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < n_chunks;
       c += int64_t(gridDim.x) * blockDim.x) {
    const int32_t k0 = first[c], k1 = first[c + 1];
    const int32_t q0 = cl_off[k0];
    desc[2 * c] = make_int4(k0, k1 - k0, q0, cl_off[k1] - q0);
    desc[2 * c + 1] = make_int4(int(wcs[k1] - wcs[k0]), 0, 0, 0);
  }
}

// Per cluster: {first row - chunk's q0, staged W offset, size, W stored}.
__global__ void k_cluster_meta(const int64_t* __restrict__ cst, const int64_t* __restrict__ wcs,
                               int64_t m, int64_t chunk_floats, const int32_t* __restrict__ first,
                               const int32_t* __restrict__ cl_off,
                               const uint8_t* __restrict__ cl_mode, int4* __restrict__ meta) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < m;
       k += int64_t(gridDim.x) * blockDim.x) {
    const int32_t k0 = first[cst[k] / chunk_floats];
    meta[k] = make_int4(cl_off[k] - cl_off[k0], int(wcs[k] - wcs[k0]), cl_off[k + 1] - cl_off[k],
                        int(cl_mode[k]));
  }
}

}  // namespace

size_t member_bytes() { return sizeof(Member); }

// Whether any record would put its cluster in a stored-W mode (k_aggregate's
// kSurface / kVol64: a surface record, or |g| > kG32); the build then
// reserves no W-block storage when none does (19 GB at C4).
__global__ void k_needs_stored_w(const uint8_t* __restrict__ kind, const double* __restrict__ g,
                                 int64_t n, int32_t* __restrict__ flag) {
  bool any = false;
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x)
    any |= kind[r] != 0 || fabs(g[r]) > double(kG32);
  if (__any_sync(0xFFFFFFFFu, any) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

void launch_needs_stored_w(const vpg_records& rec, int32_t* flag, cudaStream_t s) {
  VPG_CUDA(cudaMemsetAsync(flag, 0, sizeof(int32_t), s));
  if (rec.n > 0)
    VPG_LAUNCH(k_needs_stored_w, grid_for(rec.n, 256), 256, 0, s, rec.kind, rec.g, rec.n, flag);
}

void alloc_operator_buffers(vpg_graph* g, int64_t wt_capacity, cudaStream_t s) {
  const int64_t n = g->n;
  g->wt.alloc(size_t(wt_capacity > 0 ? wt_capacity : 1), s);
  g->phat.alloc(size_t(3 * n + 1), s);
  for (auto* v : {&g->dbar, &g->coeff, &g->acc[0], &g->acc[1]}) v->alloc(size_t(n + 1), s);
  // I vectors carry the halo slots after the n rows
  for (auto* v : {&g->i0, &g->ibuf[0], &g->ibuf[1]}) v->alloc(size_t(n + g->n_halo + 1), s);
  g->rows.alloc(size_t(4 * n + 4), s);
  g->cl_mode.alloc(size_t(n + 1), s);
  g->term_max.alloc(4, s);
  VPG_CUDA(cudaMemsetAsync(g->term_max.get(), 0, 4 * sizeof(float), s));
}

void pack_members(vpg_graph* g, const vpg_records& rec, const int32_t* list, int64_t list_n,
                  int64_t off, void* members, cudaStream_t s, const uint8_t* has_child) {
  if (list_n <= 0) return;
  // one record per thread (not a persistent grid): short blocks, so the
  // high-priority staging kernels on the side streams interleave at once
  VPG_LAUNCH(k_pack_members, grid_for(list_n, 256, 1 << 30), 256, 0, s, rec, g->clpos.get(), list, list_n,
             off, static_cast<Member*>(members), g->term_max.get(), has_child, g->i0.get());
}

void aggregate_range(vpg_graph* g, const void* members, const int64_t* range, int64_t max_count,
                     int S, cudaStream_t s) {
  if (max_count <= 0) return;
  const size_t smem = (size_t(19) * S + (S + 1) / 2) * sizeof(double);
  VPG_REQUIRE(smem <= kAggSmemMax, VPG_ELIMIT,
              "clusters larger than 160 members (cluster_size > 80) are not supported");
  ensure_dynamic_smem(reinterpret_cast<const void*>(k_aggregate), kAggSmemMax);
  const int64_t blocks = std::min<int64_t>(max_count, int64_t(sm_count()) * 16);
  VPG_LAUNCH(k_aggregate, int(blocks), kAggThreads, smem, s, static_cast<const Member*>(members),
             g->cl_off.get(), g->cl_size.get(), g->w_off.get(), range, g->n, S, g->wt.get(),
             g->phat.get(), g->dbar.get(), g->coeff.get(), g->rows.get(), g->cl_mode.get());
}

void link_children(vpg_graph* g, const vpg_records& rec, const int32_t* list, int64_t list_n,
                   cudaStream_t s) {
  if (list_n <= 0) return;
  VPG_LAUNCH(k_child_links, grid_for(list_n, 256), 256, 0, s, rec, g->clpos.get(), list, list_n,
             g->rows.get());
}

void finalize_operators_async(vpg_graph* g, const vpg_records& rec, cudaStream_t s,
                              const int32_t* parent, bool linked) {
  const int64_t n = g->n, m = g->m;
  if (n == 0) return;
  if (parent)
    VPG_LAUNCH(k_set_parents, grid_for(n, 256), 256, 0, s, parent, n, g->rows.get());
  else if (!linked)
    VPG_LAUNCH(k_parent_links, grid_for(n, 256), 256, 0, s, rec, g->clpos.get(), g->rows.get());
  // solve chunks: cost prefix over the clusters (internal order)
  int64_t* cost = scratch_of<int64_t>(s, "chunk_cost", size_t(m) + 1);
  int64_t* cst = scratch_of<int64_t>(s, "chunk_cst", size_t(m) + 1);
  int64_t* wcost = scratch_of<int64_t>(s, "chunk_wcost", size_t(m) + 1);
  int64_t* wcs = scratch_of<int64_t>(s, "chunk_wcs", size_t(m) + 1);
  VPG_LAUNCH(k_chunk_cost, grid_for(m + 1, 256), 256, 0, s, g->cl_off.get(), g->cl_mode.get(), m,
             cost, wcost);
  size_t bytes = 0;
  VPG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cost, cst, int(m + 1), s));
  void* tmp = scratch(s, "cub_temp", bytes + 256);
  VPG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, cost, cst, int(m + 1), s));
  VPG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, wcost, wcs, int(m + 1), s));
  count_launch(2);
}

void finalize_chunks(vpg_graph* g, cudaStream_t s) {
  const int64_t m = g->m, n = g->n;
  // the largest chunk (<= kChunkFloatsMax) with which 3, else 2, else 1
  // stages of chunk + the largest cluster's table, blocks and rows fit
  const int64_t smax = std::max<int64_t>(1, g->max_cluster);
  const int64_t extra = ((smax * smax + 3) & ~int64_t(3)) + kRowFloats * smax + 4;
  g->n_stages = 0;
  for (int st = 3; st >= 1 && !g->n_stages; --st) {
    const int64_t room = int64_t((kSolveSmem - 128) / (sizeof(float) * st)) - extra;
    if (room >= kChunkFloatsMin) {
      g->n_stages = st;
      g->chunk_floats = int32_t(std::min<int64_t>(kChunkFloatsMax, room & ~int64_t(3)));
    }
  }
  VPG_REQUIRE(g->n_stages > 0, VPG_ELIMIT, "clusters too large for the staged solve");
  // sum over clusters of pad4(s^2) + kRowFloats s + 4 <= smax n + kRowFloats n + 7 m
  const int64_t bound = smax * n + kRowFloats * n + 7 * m;
  g->chunk_cap = bound / g->chunk_floats + 2;
  g->chunk_first.alloc(size_t(g->chunk_cap + 1), s);
  g->chunk_desc.alloc(size_t(2 * g->chunk_cap + 2), s);
  g->cl_meta.alloc(size_t(m + 1), s);
  g->n_chunks_dev.alloc(1, s);
  if (n == 0) {
    VPG_CUDA(cudaMemsetAsync(g->chunk_first.get(), 0, sizeof(int32_t), s));
    VPG_CUDA(cudaMemsetAsync(g->n_chunks_dev.get(), 0, sizeof(int64_t), s));
    return;
  }
  const int64_t* cst = scratch_of<int64_t>(s, "chunk_cst", size_t(m) + 1);
  const int64_t* wcs = scratch_of<int64_t>(s, "chunk_wcs", size_t(m) + 1);
  VPG_LAUNCH(k_chunk_first, grid_for(g->chunk_cap + 1, 256), 256, 0, s, cst, m, g->chunk_cap,
             int64_t(g->chunk_floats), g->chunk_first.get(), g->n_chunks_dev.get());
  VPG_LAUNCH(k_chunk_desc, grid_for(g->chunk_cap, 256), 256, 0, s, g->chunk_first.get(),
             g->n_chunks_dev.get(), g->cl_off.get(), wcs, g->chunk_desc.get());
  VPG_LAUNCH(k_cluster_meta, grid_for(m, 256), 256, 0, s, cst, wcs, m, int64_t(g->chunk_floats),
             g->chunk_first.get(), g->cl_off.get(), g->cl_mode.get(), g->cl_meta.get());
}

struct PadSquare {  // a cluster's padded kernel block, pad4(s^2) floats
  __host__ __device__ int64_t operator()(int32_t sz) const {
    return (int64_t(sz) * sz + 3) & ~int64_t(3);
  }
};
struct Square {
  __host__ __device__ int64_t operator()(int32_t sz) const { return int64_t(sz) * sz; }
};
struct Widen {
  __host__ __device__ int64_t operator()(int32_t sz) const { return int64_t(sz); }
};

void build_local(vpg_graph* g, const vpg_records& rec, int64_t m, const int32_t* cl_size_host,
                 const int32_t* parent, const uint8_t* has_child, int64_t n_halo,
                 const double* halo_ipt, cudaStream_t s) {
  const int64_t n = rec.n;
  VPG_REQUIRE(n < (int64_t(1) << 31) - 1 && n_halo >= 0 && n + n_halo < (int64_t(1) << 31) - 1,
              VPG_ELIMIT, "more than 2^31-2 rows per shard");
  VPG_REQUIRE(m >= 0 && (m > 0 || n == 0), VPG_EINVAL, "cluster count does not cover the rows");
  g->n = n;
  g->m = m;
  g->n_halo = n_halo;
  // cluster geometry on the device from the sizes: offsets, padded
  // kernel-block offsets, nnz, the largest and smallest cluster
  g->cl_off.alloc(m + 1, s);
  g->cl_size.alloc(m + 1, s);
  g->w_off.alloc(m + 1, s);
  VPG_CUDA(cudaMemsetAsync(g->cl_size.get(), 0, sizeof(int32_t) * (m + 1), s));
  if (m > 0)
    VPG_CUDA(cudaMemcpyAsync(g->cl_size.get(), cl_size_host, sizeof(int32_t) * m,
                             cudaMemcpyHostToDevice, s));
  count_transfer(4 * m, 0);
  int64_t* geo = scratch_of<int64_t>(s, "local_geometry", 8);  // nnz, smax, smin
  {
    const int32_t* sz = g->cl_size.get();
    cub::TransformInputIterator<int64_t, PadSquare, const int32_t*> pads(sz, PadSquare{});
    cub::TransformInputIterator<int64_t, Square, const int32_t*> sqs(sz, Square{});
    cub::TransformInputIterator<int64_t, Widen, const int32_t*> wide(sz, Widen{});
    size_t b0 = 0, b1 = 0, b2 = 0, b3 = 0, b4 = 0;
    VPG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b0, sz, g->cl_off.get(), int(m + 1), s));
    VPG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b1, pads, g->w_off.get(), int(m + 1), s));
    VPG_CUDA(cub::DeviceReduce::Sum(nullptr, b2, sqs, geo, int(std::max<int64_t>(m, 1)), s));
    VPG_CUDA(cub::DeviceReduce::Max(nullptr, b3, wide, geo + 1, int(std::max<int64_t>(m, 1)), s));
    VPG_CUDA(cub::DeviceReduce::Min(nullptr, b4, wide, geo + 2, int(std::max<int64_t>(m, 1)), s));
    const size_t bytes = std::max({b0, b1, b2, b3, b4});
    void* tmp = scratch(s, "cub_temp", bytes + 256);
    VPG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, b0, sz, g->cl_off.get(), int(m + 1), s));
    VPG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, b1, pads, g->w_off.get(), int(m + 1), s));
    if (m > 0) {
      VPG_CUDA(cub::DeviceReduce::Sum(tmp, b2, sqs, geo, int(m), s));
      VPG_CUDA(cub::DeviceReduce::Max(tmp, b3, wide, geo + 1, int(m), s));
      VPG_CUDA(cub::DeviceReduce::Min(tmp, b4, wide, geo + 2, int(m), s));
    } else {
      VPG_CUDA(cudaMemsetAsync(geo, 0, 3 * sizeof(int64_t), s));
    }
    count_launch(5);
  }
  int64_t h_geo[3] = {0, 0, 0};
  int32_t h_total = 0;
  int64_t h_w = 0;
  VPG_CUDA(cudaMemcpyAsync(h_geo, geo, sizeof(h_geo), cudaMemcpyDeviceToHost, s));
  VPG_CUDA(cudaMemcpyAsync(&h_total, g->cl_off.get() + m, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  VPG_CUDA(cudaMemcpyAsync(&h_w, g->w_off.get() + m, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  count_transfer(0, sizeof(h_geo) + 12);
  VPG_CUDA(cudaStreamSynchronize(s));
  VPG_REQUIRE(m == 0 || h_geo[2] >= 1, VPG_EINVAL, "empty cluster in a shard-local partition");
  VPG_REQUIRE(int64_t(h_total) == n, VPG_EINVAL, "cluster sizes do not sum to the shard's row count");
  const int64_t nnz = h_geo[0], w = h_w;
  const int32_t smax = int32_t(h_geo[1]);
  g->nnz = nnz;
  g->wt_len = w;
  g->max_cluster = smax;
  g->info.n_records = n;
  g->info.n_clusters = m;
  g->info.nnz = nnz;
  g->K = std::max(1, (smax + 1) / 2);
  const int block = 256;
  g->perm.alloc(n + 1, s);
  g->clpos.alloc(n + 1, s);
  g->cluster_id.alloc(n + 1, s);
  for (auto* v : {&g->cl_center, &g->ref_of, &g->internal_of}) v->alloc(m + 1, s);
  if (n > 0) {
    VPG_LAUNCH(k_iota32, grid_for(n, block), block, 0, s, g->perm.get(), n);
    VPG_LAUNCH(k_iota32, grid_for(n, block), block, 0, s, g->clpos.get(), n);
  }
  if (m > 0) {
    VPG_LAUNCH(k_iota32, grid_for(m, block), block, 0, s, g->ref_of.get(), m);
    VPG_LAUNCH(k_iota32, grid_for(m, block), block, 0, s, g->internal_of.get(), m);
    VPG_CUDA(cudaMemsetAsync(g->cl_center.get(), 0xFF, sizeof(int32_t) * m, s));  // unknown here
    VPG_LAUNCH(k_cluster_of_rows, grid_for(m, block), block, 0, s, g->cl_off.get(), m,
               g->cluster_id.get());
  }
  // W-block storage only when some record can need a stored block (as in
  // the single-GPU build)
  int32_t needs_w = 0;
  if (n > 0) {
    int32_t* flag = scratch_of<int32_t>(s, "needs_w", 1);
    launch_needs_stored_w(rec, flag, s);
    VPG_CUDA(cudaMemcpyAsync(&needs_w, flag, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    count_transfer(0, sizeof(int32_t));
    VPG_CUDA(cudaStreamSynchronize(s));
  }
  alloc_operator_buffers(g, needs_w ? std::max<int64_t>(w, 1) : 16, s);
  if (n > 0) {
    void* members = scratch(s, "members", member_bytes() * size_t(n) + 256);
    pack_members(g, rec, nullptr, n, 0, members, s, has_child);
    DBuf<int64_t> range(2, s);
    const int64_t r[2] = {0, m};
    VPG_CUDA(cudaMemcpyAsync(range.get(), r, sizeof(r), cudaMemcpyHostToDevice, s));
    aggregate_range(g, members, range.get(), m, std::max(1, int(smax)), s);
    if (n_halo > 0)
      VPG_LAUNCH(k_halo_i0, grid_for(n_halo, block), block, 0, s, halo_ipt, n_halo,
                 g->i0.get() + n);
  }
  finalize_operators_async(g, rec, s, parent);
  VPG_CUDA(cudaStreamSynchronize(s));
  finalize_chunks(g, s);
  VPG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace vpg

// Aggregation operators, the device-resident fixed-point solve, and the splat.
//
//   k_operators   compute_marginals (graph.py:94-120) + _build_operators
//                 (graph.py:123-168): per cluster, p-hat for every member
//                 sample, the s x s kernel block W (stored transposed, fp32),
//                 D-bar, and the per-row solve vectors.  fp64 arithmetic
//                 (HG at g >= 0.9 needs it), numpy's rounding
//                 order for dot products.
//   k_iterate     one fixed-point iteration (solve.py:78-83): block-dense
//                 W*I per cluster, propagation along the continuation edge
//                 (operators.py:41-47) fused as a scatter into the parent
//                 row, and the residual maxima (solve.py:54-61).
//   k_control     residual, tol break and 3-growth divergence (solve.py:80-94)
//                 evaluated on the device so the loop never syncs the host.
//   k_splat       splat_output (solve.py:101-132).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.cuh"

namespace vpg {
namespace {

constexpr double kInv4Pi = 1.0 / (4.0 * 3.14159265358979323846);
constexpr double kInvPi = 1.0 / 3.14159265358979323846;
constexpr int kWarpCap = 64;  // members staged per warp in shared memory
constexpr int kOpWarps = 4;   // warps per block in k_operators
constexpr int kItWarps = 8;   // warps per block in k_iterate

// numpy's einsum order for a length-3 contraction, no FMA.
__device__ __forceinline__ double dot3(double ax, double ay, double az, double bx, double by,
                                       double bz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(ax, bx), __dmul_rn(ay, by)), __dmul_rn(az, bz));
}

// Member cache in shared memory (structure of arrays, one warp's cluster).
struct MemberCache {
  double ax[kWarpCap], ay[kWarpCap], az[kWarpCap];  // -omega_out (volume) or normal
  double px[kWarpCap], py[kWarpCap], pz[kWarpCap];  // phase_dir
  double ex[kWarpCap], ey[kWarpCap], ez[kWarpCap];  // emit_dir
  double num[kWarpCap], c1[kWarpCap], c2[kWarpCap]; // HG: INV4PI(1-g^2), 1+g^2, 2g
  double inv_p[kWarpCap];                            // 1/phat_ind or 0 (excluded)
  double wex[kWarpCap], wey[kWarpCap], wez[kWarpCap];  // d_emit / phat_dir_emit
  double wpx[kWarpCap], wpy[kWarpCap], wpz[kWarpCap];  // d_phase / phat_dir_phase
};

// Member l's strategy density toward direction d (graph.py:82-91).
__device__ __forceinline__ double strategy_pdf(const MemberCache& c, int l, bool volume,
                                               double dx, double dy, double dz) {
  const double cs = dot3(c.ax[l], c.ay[l], c.az[l], dx, dy, dz);
  if (!volume) return cs > 0.0 ? __dmul_rn(cs, kInvPi) : 0.0;
  const double den = __dsub_rn(c.c1[l], __dmul_rn(c.c2[l], cs));
  return __ddiv_rn(c.num[l], __dmul_rn(den, __dsqrt_rn(den)));
}

__device__ __forceinline__ double hg_pdf(double cs, double g) {
  const double g2 = __dmul_rn(g, g);
  const double den = __dsub_rn(__dadd_rn(1.0, g2), __dmul_rn(__dmul_rn(2.0, g), cs));
  return __ddiv_rn(__dmul_rn(kInv4Pi, __dsub_rn(1.0, g2)), __dmul_rn(den, __dsqrt_rn(den)));
}

__device__ __forceinline__ float4 f4(double x, double y, double z) {
  return make_float4(float(x), float(y), float(z), 0.f);
}

__device__ __forceinline__ void atomic_max_pos(float* addr, float v) {
  // v >= 0: the IEEE bit pattern orders like the value
  atomicMax(reinterpret_cast<unsigned int*>(addr), __float_as_uint(v));
}

// One warp per cluster (s <= kWarpCap).
__global__ void __launch_bounds__(kOpWarps * 32)
k_operators(vpg_records rec, const int32_t* __restrict__ perm, const int32_t* __restrict__ clpos,
            const int32_t* __restrict__ cl_off, const int64_t* __restrict__ w_off, int64_t m,
            int64_t n, float* __restrict__ wt, double* __restrict__ phat,
            float4* __restrict__ dbar_o, float4* __restrict__ coeff_o, float4* __restrict__ a_o,
            float4* __restrict__ b_o, float4* __restrict__ i0_o, int32_t* __restrict__ par_o,
            float* __restrict__ term_max) {
  __shared__ MemberCache cache[kOpWarps];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  MemberCache& c = cache[wid];
  const int64_t nwarps = int64_t(gridDim.x) * kOpWarps;
  float tmax[3] = {0.f, 0.f, 0.f};

  for (int64_t k = int64_t(blockIdx.x) * kOpWarps + wid; k < m; k += nwarps) {
    const int32_t q0 = cl_off[k];
    const int s = cl_off[k + 1] - q0;
    const int64_t wb = w_off[k];
    const bool volume = rec.kind[perm[q0]] == 0;
    const double ks = double(s);

    // stage member geometry
    for (int l = lane; l < s; l += 32) {
      const int64_t r = perm[q0 + l];
      if (volume) {
        c.ax[l] = -rec.omega_out[r * 3];
        c.ay[l] = -rec.omega_out[r * 3 + 1];
        c.az[l] = -rec.omega_out[r * 3 + 2];
        const double g = rec.g[r];
        const double g2 = __dmul_rn(g, g);
        c.num[l] = __dmul_rn(kInv4Pi, __dsub_rn(1.0, g2));
        c.c1[l] = __dadd_rn(1.0, g2);
        c.c2[l] = __dmul_rn(2.0, g);
      } else {
        c.ax[l] = rec.normal[r * 3];
        c.ay[l] = rec.normal[r * 3 + 1];
        c.az[l] = rec.normal[r * 3 + 2];
      }
      c.px[l] = rec.phase_dir[r * 3];
      c.py[l] = rec.phase_dir[r * 3 + 1];
      c.pz[l] = rec.phase_dir[r * 3 + 2];
      c.ex[l] = rec.emit_dir[r * 3];
      c.ey[l] = rec.emit_dir[r * 3 + 1];
      c.ez[l] = rec.emit_dir[r * 3 + 2];
    }
    __syncwarp();

    // pass 1: marginals of every member sample (column j)
    for (int j = lane; j < s; j += 32) {
      const int64_t r = perm[q0 + j];
      double sp = 0.0, se = 0.0;
      for (int l = 0; l < s; ++l) {
        sp = __dadd_rn(sp, strategy_pdf(c, l, volume, c.px[j], c.py[j], c.pz[j]));
        se = __dadd_rn(se, strategy_pdf(c, l, volume, c.ex[j], c.ey[j], c.ez[j]));
      }
      const double p_ind = sp;
      const double p_dp = __dadd_rn(sp, __dmul_rn(ks, rec.pdf_emit_at_phase[r]));
      const double p_de = rec.emit_delta[r] ? ks : __dadd_rn(se, __dmul_rn(ks, rec.pdf_emit[r]));
      const int64_t q = q0 + j;
      phat[q] = p_ind;
      phat[n + q] = p_dp;
      phat[2 * n + q] = p_de;
      const bool inc_p = isfinite(p_ind) && p_ind > 0.0;
      const bool inc_e = isfinite(p_de) && p_de > 0.0;
      const bool ok_dp = inc_p && isfinite(p_dp) && p_dp > 0.0;
      c.inv_p[j] = inc_p ? __ddiv_rn(1.0, p_ind) : 0.0;
      const double ie = inc_e ? __ddiv_rn(1.0, p_de) : 0.0;
      const double ip = ok_dp ? __ddiv_rn(1.0, p_dp) : 0.0;
      c.wex[j] = rec.d_emit[r * 3] * ie;
      c.wey[j] = rec.d_emit[r * 3 + 1] * ie;
      c.wez[j] = rec.d_emit[r * 3 + 2] * ie;
      c.wpx[j] = rec.d_phase[r * 3] * ip;
      c.wpy[j] = rec.d_phase[r * 3 + 1] * ip;
      c.wpz[j] = rec.d_phase[r * 3 + 2] * ip;
    }
    __syncwarp();

    // pass 2: kernel rows, D-bar and solve vectors (row rr)
    for (int rr = lane; rr < s; rr += 32) {
      const int64_t r = perm[q0 + rr];
      double dx = 0.0, dy = 0.0, dz = 0.0;
      for (int j = 0; j < s; ++j) {
        const double pd = strategy_pdf(c, rr, volume, c.px[j], c.py[j], c.pz[j]);
        const double pe = strategy_pdf(c, rr, volume, c.ex[j], c.ey[j], c.ez[j]);
        wt[wb + int64_t(j) * s + rr] = float(pd * c.inv_p[j]);
        dx += pe * c.wex[j] + pd * c.wpx[j];
        dy += pe * c.wey[j] + pd * c.wpy[j];
        dz += pe * c.wez[j] + pd * c.wpz[j];
      }
      const double kx = rec.coeff[r * 3], ky = rec.coeff[r * 3 + 1], kz = rec.coeff[r * 3 + 2];
      const double wx = rec.w_cont[r * 3], wy = rec.w_cont[r * 3 + 1], wz = rec.w_cont[r * 3 + 2];
      const double bx = kx * dx, by = ky * dy, bz = kz * dz;
      const int64_t q = q0 + rr;
      dbar_o[q] = f4(bx, by, bz);
      coeff_o[q] = f4(kx, ky, kz);
      a_o[q] = f4(wx * kx, wy * ky, wz * kz);
      b_o[q] = f4(wx * bx, wy * by, wz * bz);
      const double ix = rec.i_pt[r * 3], iy = rec.i_pt[r * 3 + 1], iz = rec.i_pt[r * 3 + 2];
      i0_o[q] = f4(ix, iy, iz);
      const int64_t pid = rec.path_idx[r];
      par_o[q] = (r > 0 && rec.path_idx[r - 1] == pid) ? clpos[r - 1] : -1;
      const bool terminal = !(r + 1 < n && rec.path_idx[r + 1] == pid);
      if (terminal) {
        tmax[0] = fmaxf(tmax[0], fabsf(float(ix)));
        tmax[1] = fmaxf(tmax[1], fabsf(float(iy)));
        tmax[2] = fmaxf(tmax[2], fabsf(float(iz)));
      }
    }
    __syncwarp();
  }
  for (int ch = 0; ch < 3; ++ch) {
    float v = tmax[ch];
    for (int off = 16; off; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, off));
    if (lane == 0 && v > 0.f) atomic_max_pos(&term_max[ch], v);
  }
}

// One fixed-point iteration t; mode 0 = solve step, 1 = aggregate only.
// Warp per cluster; rows and columns processed in chunks of 64.
template <int kMode>
__global__ void __launch_bounds__(kItWarps * 32)
k_iterate(const int32_t* __restrict__ cl_off, const int64_t* __restrict__ w_off, int64_t m,
          const float* __restrict__ wt, const float4* __restrict__ i_in,
          float4* __restrict__ i_out, const float4* __restrict__ acc_prev,
          float4* __restrict__ acc_out, const float4* __restrict__ av,
          const float4* __restrict__ bv, const float4* __restrict__ i0,
          const int32_t* __restrict__ par, int t, uint32_t* __restrict__ red,
          const int32_t* __restrict__ ctl) {
  if (kMode == 0 && ctl[1]) return;  // converged or diverged earlier
  __shared__ float4 stage[kItWarps][kWarpCap];
  __shared__ float blk[kItWarps][6];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int64_t nwarps = int64_t(gridDim.x) * kItWarps;
  float dmax[3] = {0.f, 0.f, 0.f}, smax[3] = {0.f, 0.f, 0.f};
  unsigned nan_bits = 0;  // numpy's max propagates NaN per channel: remember it

  for (int64_t k = int64_t(blockIdx.x) * kItWarps + wid; k < m; k += nwarps) {
    const int32_t q0 = cl_off[k];
    const int s = cl_off[k + 1] - q0;
    const float* w = wt + w_off[k];
    for (int rc = 0; rc < s; rc += 64) {
      const int r0 = rc + lane, r1 = rc + lane + 32;
      float3 acc0 = make_float3(0.f, 0.f, 0.f), acc1 = acc0;
      for (int cc = 0; cc < s; cc += kWarpCap) {
        const int cn = min(kWarpCap, s - cc);
        if (lane < cn) stage[wid][lane] = i_in[q0 + cc + lane];
        if (lane + 32 < cn) stage[wid][lane + 32] = i_in[q0 + cc + lane + 32];
        __syncwarp();
#pragma unroll 4
        for (int j = 0; j < cn; ++j) {
          const float4 ij = stage[wid][j];
          const float* col = w + int64_t(cc + j) * s;
          const float w0 = r0 < s ? __ldg(col + r0) : 0.f;
          const float w1 = r1 < s ? __ldg(col + r1) : 0.f;
          acc0.x = fmaf(w0, ij.x, acc0.x);
          acc0.y = fmaf(w0, ij.y, acc0.y);
          acc0.z = fmaf(w0, ij.z, acc0.z);
          acc1.x = fmaf(w1, ij.x, acc1.x);
          acc1.y = fmaf(w1, ij.y, acc1.y);
          acc1.z = fmaf(w1, ij.z, acc1.z);
        }
        __syncwarp();
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rr = h ? r1 : r0;
        if (rr >= s) continue;
        const float3 ac = h ? acc1 : acc0;
        const int64_t q = q0 + rr;
        acc_out[q] = make_float4(ac.x, ac.y, ac.z, 0.f);
        if (kMode != 0) continue;
        const int32_t p = par[q];
        if (p < 0) continue;
        const float4 A = av[q], B = bv[q];
        const float nx = fmaf(A.x, ac.x, B.x), ny = fmaf(A.y, ac.y, B.y), nz = fmaf(A.z, ac.z, B.z);
        float4 old;
        if (t == 0) {
          old = i0[p];
        } else {
          const float4 pa = acc_prev[q];
          old = make_float4(fmaf(A.x, pa.x, B.x), fmaf(A.y, pa.y, B.y), fmaf(A.z, pa.z, B.z), 0.f);
        }
        i_out[p] = make_float4(nx, ny, nz, 0.f);
        const float dv[3] = {fabsf(nx - old.x), fabsf(ny - old.y), fabsf(nz - old.z)};
        const float sv[3] = {fabsf(nx), fabsf(ny), fabsf(nz)};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (dv[c] != dv[c]) nan_bits |= 1u << c;
          if (sv[c] != sv[c]) nan_bits |= 8u << c;
          dmax[c] = fmaxf(dmax[c], dv[c]);
          smax[c] = fmaxf(smax[c], sv[c]);
        }
      }
    }
  }
  if (kMode != 0) return;
  for (int off = 16; off; off >>= 1) nan_bits |= __shfl_xor_sync(0xFFFFFFFFu, nan_bits, off);
  if (lane == 0 && nan_bits) atomicOr(&red[t * 8 + 6], nan_bits);
  float v[6] = {dmax[0], dmax[1], dmax[2], smax[0], smax[1], smax[2]};
#pragma unroll
  for (int i = 0; i < 6; ++i)
    for (int off = 16; off; off >>= 1) v[i] = fmaxf(v[i], __shfl_xor_sync(0xFFFFFFFFu, v[i], off));
  if (lane == 0)
    for (int i = 0; i < 6; ++i) blk[wid][i] = v[i];
  __syncthreads();
  if (threadIdx.x < 6) {
    float x = 0.f;
    for (int w2 = 0; w2 < kItWarps; ++w2) x = fmaxf(x, blk[w2][threadIdx.x]);
    if (x > 0.f) atomicMax(&red[t * 8 + threadIdx.x], __float_as_uint(x));
  }
}

// Residual bookkeeping for iteration t (solve.py:54-61,80-94).
// ctl = {performed, stop, grow, diverged}
__global__ void k_control(int t, double tol, const uint32_t* __restrict__ red,
                          const float* __restrict__ term_max, double* __restrict__ resid,
                          int32_t* __restrict__ ctl) {
  if (threadIdx.x != 0 || ctl[1]) return;
  const unsigned nan_bits = red[t * 8 + 6];
  double worst = 0.0;
  for (int c = 0; c < 3; ++c) {
    // a NaN channel never wins Python's max(worst, q) in the reference
    if (nan_bits & ((1u | 8u) << c)) continue;
    const double delta = double(__uint_as_float(red[t * 8 + c]));
    double scale = double(fmaxf(__uint_as_float(red[t * 8 + 3 + c]), term_max[c]));
    scale = scale > 1e-12 ? scale : 1e-12;
    const double q = delta / scale;
    worst = q > worst ? q : worst;
  }
  resid[t] = worst;
  ctl[0] = t + 1;
  if (t >= 1 && worst > resid[t - 1]) {
    ctl[2] += 1;
    if (ctl[2] >= 3) {
      ctl[3] = 1;
      ctl[1] = 1;
      return;
    }
  } else {
    ctl[2] = 0;
  }
  if (worst < tol) ctl[1] = 1;
}

// Single-strategy I-bar / coeff (the 0-iteration result, solve.py:41-51).
__global__ void k_own_indirect(vpg_records rec, const int32_t* __restrict__ perm, int64_t n,
                               float4* __restrict__ acc_out) {
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < n;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = perm[q];
    const double dx = rec.phase_dir[r * 3], dy = rec.phase_dir[r * 3 + 1], dz = rec.phase_dir[r * 3 + 2];
    double rho;
    if (rec.kind[r] == 0) {
      rho = hg_pdf(dot3(-rec.omega_out[r * 3], -rec.omega_out[r * 3 + 1], -rec.omega_out[r * 3 + 2],
                        dx, dy, dz), rec.g[r]);
    } else {
      const double cs = dot3(rec.normal[r * 3], rec.normal[r * 3 + 1], rec.normal[r * 3 + 2], dx, dy, dz);
      rho = (cs > 0.0 ? cs : 0.0) / 3.14159265358979323846;
    }
    const double pp = rec.pdf_phase[r];
    const double ratio = pp > 0.0 ? rho / pp : 0.0;
    acc_out[q] = f4(ratio * rec.i_pt[r * 3], ratio * rec.i_pt[r * 3 + 1], ratio * rec.i_pt[r * 3 + 2]);
  }
}

__global__ void k_fill_f4(float4* __restrict__ dst, const float4* __restrict__ src, int64_t n) {
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < n;
       q += int64_t(gridDim.x) * blockDim.x)
    dst[q] = src[q];
}

// Record-order fp64 (n,3) <-> cluster-major float4.
__global__ void k_gather_rec3(const double* __restrict__ src, const int32_t* __restrict__ perm,
                              int64_t n, float4* __restrict__ dst) {
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < n;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = perm[q];
    dst[q] = f4(src[r * 3], src[r * 3 + 1], src[r * 3 + 2]);
  }
}

// out[r] = scale[r] (fp64, optional) * v[clpos[r]]
__global__ void k_scatter_rec3(const float4* __restrict__ v, const int32_t* __restrict__ clpos,
                               const double* __restrict__ scale, int64_t n, double* __restrict__ out) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const float4 x = v[clpos[r]];
    if (scale) {
      out[r * 3] = scale[r * 3] * double(x.x);
      out[r * 3 + 1] = scale[r * 3 + 1] * double(x.y);
      out[r * 3 + 2] = scale[r * 3 + 2] * double(x.z);
    } else {
      out[r * 3] = x.x;
      out[r * 3 + 1] = x.y;
      out[r * 3 + 2] = x.z;
    }
  }
}

__global__ void k_scatter_phat(const double* __restrict__ phat, const int32_t* __restrict__ clpos,
                               int64_t n, double* __restrict__ o0, double* __restrict__ o1,
                               double* __restrict__ o2) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t q = clpos[r];
    o0[r] = phat[q];
    o1[r] = phat[n + q];
    o2[r] = phat[2 * n + q];
  }
}

__global__ void k_row_sizes(const int32_t* __restrict__ cluster_id, const int32_t* __restrict__ cl_off,
                            int64_t n, int64_t* __restrict__ sz) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r <= n;
       r += int64_t(gridDim.x) * blockDim.x) {
    if (r == n) { sz[r] = 0; continue; }
    const int32_t k = cluster_id[r];
    sz[r] = cl_off[k + 1] - cl_off[k];
  }
}

// CSR rows of W in record order (graph.py:167): warp per row.
__global__ void k_export_csr(const int32_t* __restrict__ cluster_id, const int32_t* __restrict__ clpos,
                             const int32_t* __restrict__ cl_off, const int64_t* __restrict__ w_off,
                             const int32_t* __restrict__ perm, const float* __restrict__ wt,
                             const int64_t* __restrict__ indptr, int64_t n,
                             int64_t* __restrict__ indices, double* __restrict__ data) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; r < n; r += nwarps) {
    const int32_t k = cluster_id[r];
    const int32_t q0 = cl_off[k];
    const int s = cl_off[k + 1] - q0;
    const int rl = clpos[r] - q0;
    const int64_t base = indptr[r];
    for (int j = lane; j < s; j += 32) {
      indices[base + j] = perm[q0 + j];
      data[base + j] = double(wt[w_off[k] + int64_t(j) * s + rl]);
    }
  }
}

__global__ void k_i32_to_i64(const int32_t* __restrict__ a, int64_t n, int64_t* __restrict__ b) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    b[i] = a[i];
}

// propagate / propagate_linear (operators.py:27-47), record order, fp64.
__global__ void k_propagate(vpg_records rec, const double* __restrict__ lbar, int linear,
                            double* __restrict__ out) {
  const int64_t n = rec.n;
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const bool child = r + 1 < n && rec.path_idx[r + 1] == rec.path_idx[r];
    for (int c = 0; c < 3; ++c) {
      double v;
      if (child) v = rec.w_cont[(r + 1) * 3 + c] * lbar[(r + 1) * 3 + c];
      else v = linear ? 0.0 : rec.i_pt[r * 3 + c];
      out[r * 3 + c] = v;
    }
  }
}

// splat_output (solve.py:101-132): thread per pixel, samples in order.
__global__ void k_splat(vpg_paths P, const double* __restrict__ coeff, const int32_t* __restrict__ clpos,
                        const float4* __restrict__ acc, const float4* __restrict__ dbar,
                        int64_t npix, int spp, int mode, double* __restrict__ image) {
  for (int64_t pix = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; pix < npix;
       pix += int64_t(gridDim.x) * blockDim.x) {
    double sx = 0.0, sy = 0.0, sz = 0.0;
    for (int s = 0; s < spp; ++s) {
      const int64_t p = pix * spp + s;
      double vx = P.d_cam[p * 3], vy = P.d_cam[p * 3 + 1], vz = P.d_cam[p * 3 + 2];
      if (P.rec_count[p] > 0) {
        const int64_t r0 = P.rec_start[p];
        const int64_t q = clpos[r0];
        double dx, dy, dz;
        if (mode == VPG_DIRECT_AGGREGATED) {
          const float4 d = dbar[q];
          dx = d.x; dy = d.y; dz = d.z;
        } else {
          const double* src = mode == VPG_DIRECT_EXTRA ? P.extra_direct : P.direct0;
          dx = src[p * 3]; dy = src[p * 3 + 1]; dz = src[p * 3 + 2];
        }
        const float4 ac = acc[q];
        const double ix = coeff[r0 * 3] * double(ac.x), iy = coeff[r0 * 3 + 1] * double(ac.y),
                     iz = coeff[r0 * 3 + 2] * double(ac.z);
        vx += P.cam_weight[p * 3] * (dx + ix);
        vy += P.cam_weight[p * 3 + 1] * (dy + iy);
        vz += P.cam_weight[p * 3 + 2] * (dz + iz);
      }
      sx += vx; sy += vy; sz += vz;
    }
    image[pix * 3] = sx / spp;
    image[pix * 3 + 1] = sy / spp;
    image[pix * 3 + 2] = sz / spp;
  }
}

__global__ void k_splat_pt(vpg_paths P, int64_t npix, int spp, double* __restrict__ image) {
  for (int64_t pix = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; pix < npix;
       pix += int64_t(gridDim.x) * blockDim.x) {
    double sx = 0.0, sy = 0.0, sz = 0.0;
    for (int s = 0; s < spp; ++s) {
      const int64_t p = pix * spp + s;
      sx += P.pt_estimate[p * 3];
      sy += P.pt_estimate[p * 3 + 1];
      sz += P.pt_estimate[p * 3 + 2];
    }
    image[pix * 3] = sx / spp;
    image[pix * 3 + 1] = sy / spp;
    image[pix * 3 + 2] = sz / spp;
  }
}

int iterate_grid(int64_t m) {
  int64_t blocks = (m + kItWarps - 1) / kItWarps;
  const int64_t cap = int64_t(sm_count()) * 8;
  return int(blocks < cap ? blocks : cap);
}

}  // namespace

void build_operators(vpg_graph* g, const vpg_records& rec, cudaStream_t s) {
  const int64_t n = g->n, m = g->m;
  VPG_REQUIRE(g->max_cluster <= kWarpCap, VPG_ELIMIT,
              "clusters larger than 64 members (cluster_size > 32) are not supported yet");
  g->wt.alloc(size_t(g->nnz > 0 ? g->nnz : 1), s);
  g->phat.alloc(size_t(3 * n + 1), s);
  for (auto* v : {&g->i0, &g->a, &g->b, &g->dbar, &g->coeff, &g->ibuf[0], &g->ibuf[1], &g->acc[0],
                  &g->acc[1]})
    v->alloc(size_t(n + 1), s);
  g->par.alloc(size_t(n + 1), s);
  g->term_max.alloc(4, s);
  VPG_CUDA(cudaMemsetAsync(g->term_max.get(), 0, 4 * sizeof(float), s));
  if (n == 0) return;
  int64_t blocks = (m + kOpWarps - 1) / kOpWarps;
  const int64_t cap = int64_t(sm_count()) * 16;
  VPG_LAUNCH(k_operators, int(blocks < cap ? blocks : cap), kOpWarps * 32, 0, s, rec,
             g->perm.get(), g->clpos.get(), g->cl_off.get(), g->w_off.get(), m, n, g->wt.get(),
             g->phat.get(), g->dbar.get(), g->coeff.get(), g->a.get(), g->b.get(), g->i0.get(),
             g->par.get(), g->term_max.get());
}

// ------------------------------------------------------------------ solve
void solve(vpg_graph* g, const vpg_records& rec, int32_t iterations, double tol,
           double* residuals, int32_t* performed, cudaStream_t s) {
  VPG_REQUIRE(iterations >= 0, VPG_EINVAL, "iterations must be >= 0");
  const int64_t n = g->n, m = g->m;
  if (g->red_cap < iterations + 1) {
    g->red.alloc(size_t(iterations + 1) * 8, s);
    g->resid.alloc(size_t(iterations + 1), s);
    g->red_cap = iterations + 1;
  }
  if (!g->ctl.get()) g->ctl.alloc(4, s);
  VPG_CUDA(cudaMemsetAsync(g->red.get(), 0, g->red.bytes(), s));
  VPG_CUDA(cudaMemsetAsync(g->ctl.get(), 0, 4 * sizeof(int32_t), s));
  const int block = 256;
  if (n > 0) {
    VPG_LAUNCH(k_fill_f4, grid_for(n, block), block, 0, s, g->ibuf[0].get(), g->i0.get(), n);
    VPG_LAUNCH(k_fill_f4, grid_for(n, block), block, 0, s, g->ibuf[1].get(), g->i0.get(), n);
    if (iterations == 0)
      VPG_LAUNCH(k_own_indirect, grid_for(n, block), block, 0, s, rec, g->perm.get(), n,
                 g->acc[0].get());
  }
  const int grid = iterate_grid(m);
  for (int t = 0; t < iterations && n > 0; ++t) {
    VPG_LAUNCH(k_iterate<0>, grid, kItWarps * 32, 0, s, g->cl_off.get(), g->w_off.get(), m,
               g->wt.get(), g->ibuf[t & 1].get(), g->ibuf[(t + 1) & 1].get(), g->acc[t & 1].get(),
               g->acc[(t + 1) & 1].get(), g->a.get(), g->b.get(), g->i0.get(), g->par.get(), t,
               g->red.get(), g->ctl.get());
    VPG_LAUNCH(k_control, 1, 32, 0, s, t, tol, g->red.get(), g->term_max.get(), g->resid.get(),
               g->ctl.get());
  }
  int32_t ctl_h[4] = {0, 0, 0, 0};
  if (n > 0 && iterations > 0) {
    VPG_CUDA(cudaMemcpyAsync(ctl_h, g->ctl.get(), sizeof(ctl_h), cudaMemcpyDeviceToHost, s));
    VPG_CUDA(cudaMemcpyAsync(residuals, g->resid.get(), sizeof(double) * iterations,
                             cudaMemcpyDeviceToHost, s));
    count_transfer(0, sizeof(ctl_h) + sizeof(double) * iterations);
  } else if (iterations > 0) {
    // an empty graph: every residual is 0/1e-12 = 0 and the tol test stops at once
    for (int t = 0; t < iterations; ++t) residuals[t] = 0.0;
    ctl_h[0] = tol > 0.0 ? 1 : iterations;
  }
  VPG_CUDA(cudaStreamSynchronize(s));
  g->performed = ctl_h[0];
  *performed = ctl_h[0];
  if (ctl_h[3]) throw Error(VPG_EDIVERGED, "fixed-point residuals grew over 3 consecutive iterations");
}

void solve_export(const vpg_graph* g, const vpg_records& rec, double* incoming, double* i_bar,
                  cudaStream_t s) {
  VPG_REQUIRE(g->performed >= 0, VPG_EINVAL, "solve has not run on this graph");
  const int64_t n = g->n;
  if (n == 0) return;
  const int block = 256;
  const int cur = g->performed & 1;
  DBuf<double> tmp(size_t(n) * 3, s);
  if (incoming) {
    VPG_LAUNCH(k_scatter_rec3, grid_for(n, block), block, 0, s, g->ibuf[cur].get(),
               g->clpos.get(), nullptr, n, tmp.get());
    VPG_CUDA(cudaMemcpyAsync(incoming, tmp.get(), n * 24, cudaMemcpyDeviceToHost, s));
    VPG_CUDA(cudaStreamSynchronize(s));
  }
  if (i_bar) {
    VPG_LAUNCH(k_scatter_rec3, grid_for(n, block), block, 0, s, g->acc[cur].get(),
               g->clpos.get(), rec.coeff, n, tmp.get());
    VPG_CUDA(cudaMemcpyAsync(i_bar, tmp.get(), n * 24, cudaMemcpyDeviceToHost, s));
    VPG_CUDA(cudaStreamSynchronize(s));
  }
}

void aggregate_indirect(const vpg_graph* g, const vpg_records& rec, const double* incoming,
                        double* out, cudaStream_t s) {
  const int64_t n = g->n;
  if (n == 0) return;
  const int block = 256;
  DBuf<float4> vin(n, s), vout(n, s);
  VPG_LAUNCH(k_gather_rec3, grid_for(n, block), block, 0, s, incoming, g->perm.get(), n, vin.get());
  VPG_LAUNCH(k_iterate<1>, iterate_grid(g->m), kItWarps * 32, 0, s, g->cl_off.get(),
             g->w_off.get(), g->m, g->wt.get(), vin.get(), nullptr, nullptr, vout.get(), nullptr,
             nullptr, nullptr, nullptr, 0, nullptr, nullptr);
  VPG_LAUNCH(k_scatter_rec3, grid_for(n, block), block, 0, s, vout.get(), g->clpos.get(),
             rec.coeff, n, out);
}

void propagate(const vpg_records& rec, const double* lbar, double* out, int linear,
               cudaStream_t s) {
  if (rec.n == 0) return;
  VPG_LAUNCH(k_propagate, grid_for(rec.n, 256), 256, 0, s, rec, lbar, linear, out);
}

void export_clusters(const vpg_graph* g, int64_t* cluster_id, int64_t* cl_off, int64_t* members,
                     int64_t* centers, cudaStream_t s) {
  const int64_t n = g->n, m = g->m;
  const int block = 256;
  DBuf<int64_t> tmp(size_t(std::max<int64_t>(n, m + 1)) + 1, s);
  auto out = [&](const int32_t* src, int64_t cnt, int64_t* host) {
    if (!host || cnt == 0) return;
    VPG_LAUNCH(k_i32_to_i64, grid_for(cnt, block), block, 0, s, src, cnt, tmp.get());
    VPG_CUDA(cudaMemcpyAsync(host, tmp.get(), cnt * 8, cudaMemcpyDeviceToHost, s));
    VPG_CUDA(cudaStreamSynchronize(s));
  };
  out(g->cluster_id.get(), n, cluster_id);
  out(g->cl_off.get(), m + 1, cl_off);
  out(g->perm.get(), n, members);
  out(g->cl_center.get(), m, centers);
}

void export_marginals(const vpg_graph* g, double* p0, double* p1, double* p2, cudaStream_t s) {
  const int64_t n = g->n;
  if (n == 0) return;
  DBuf<double> tmp(size_t(n) * 3, s);
  VPG_LAUNCH(k_scatter_phat, grid_for(n, 256), 256, 0, s, g->phat.get(), g->clpos.get(), n,
             tmp.get(), tmp.get() + n, tmp.get() + 2 * n);
  double* dst[3] = {p0, p1, p2};
  for (int i = 0; i < 3; ++i)
    if (dst[i]) VPG_CUDA(cudaMemcpyAsync(dst[i], tmp.get() + i * n, n * 8, cudaMemcpyDeviceToHost, s));
  VPG_CUDA(cudaStreamSynchronize(s));
}

void export_operators(const vpg_graph* g, int64_t* indptr, int64_t* indices, double* data,
                      double* d_bar, cudaStream_t s) {
  const int64_t n = g->n;
  if (n == 0) {
    if (indptr) indptr[0] = 0;
    return;
  }
  const int block = 256;
  if (indptr || indices || data) {
    DBuf<int64_t> sz(n + 1, s), ip(n + 1, s);
    VPG_LAUNCH(k_row_sizes, grid_for(n + 1, block), block, 0, s, g->cluster_id.get(),
               g->cl_off.get(), n, sz.get());
    size_t bytes = 0;
    VPG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, sz.get(), ip.get(), int(n + 1), s));
    {
      DBuf<char> t(bytes, s);
      VPG_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), bytes, sz.get(), ip.get(), int(n + 1), s));
      count_launch(1);
    }
    if (indptr) VPG_CUDA(cudaMemcpyAsync(indptr, ip.get(), (n + 1) * 8, cudaMemcpyDeviceToHost, s));
    if (indices || data) {
      DBuf<int64_t> ind(size_t(g->nnz) + 1, s);
      DBuf<double> dat(size_t(g->nnz) + 1, s);
      VPG_LAUNCH(k_export_csr, grid_for(n * 32, block), block, 0, s, g->cluster_id.get(),
                 g->clpos.get(), g->cl_off.get(), g->w_off.get(), g->perm.get(), g->wt.get(),
                 ip.get(), n, ind.get(), dat.get());
      if (indices) VPG_CUDA(cudaMemcpyAsync(indices, ind.get(), g->nnz * 8, cudaMemcpyDeviceToHost, s));
      if (data) VPG_CUDA(cudaMemcpyAsync(data, dat.get(), g->nnz * 8, cudaMemcpyDeviceToHost, s));
      VPG_CUDA(cudaStreamSynchronize(s));
    }
    VPG_CUDA(cudaStreamSynchronize(s));
  }
  if (d_bar) {
    DBuf<double> tmp(size_t(n) * 3, s);
    VPG_LAUNCH(k_scatter_rec3, grid_for(n, block), block, 0, s, g->dbar.get(), g->clpos.get(),
               nullptr, n, tmp.get());
    VPG_CUDA(cudaMemcpyAsync(d_bar, tmp.get(), n * 24, cudaMemcpyDeviceToHost, s));
    VPG_CUDA(cudaStreamSynchronize(s));
  }
}

void splat(const vpg_graph* g, const vpg_records& rec, const vpg_paths& P, int w, int h, int spp,
           int mode, double* image, cudaStream_t s) {
  VPG_REQUIRE(g->performed >= 0, VPG_EINVAL, "solve has not run on this graph");
  VPG_REQUIRE(P.n == int64_t(w) * h * spp, VPG_EINVAL, "path table size != width*height*spp");
  const int64_t npix = int64_t(w) * h;
  VPG_LAUNCH(k_splat, grid_for(npix, 128), 128, 0, s, P, rec.coeff, g->clpos.get(),
             g->acc[g->performed & 1].get(), g->dbar.get(), npix, spp, mode, image);
}

void splat_pt(const vpg_paths& P, int w, int h, int spp, double* image, cudaStream_t s) {
  VPG_REQUIRE(P.n == int64_t(w) * h * spp, VPG_EINVAL, "path table size != width*height*spp");
  const int64_t npix = int64_t(w) * h;
  VPG_LAUNCH(k_splat_pt, grid_for(npix, 128), 128, 0, s, P, npix, spp, image);
}

}  // namespace vpg

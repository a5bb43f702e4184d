// The device-resident fixed-point solve, operator application, exports and the splat.
//
//   (the operators themselves are built in aggregation.cu)
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

// numpy's einsum order for a length-3 contraction, no FMA.
__device__ __forceinline__ double dot3(double ax, double ay, double az, double bx, double by,
                                       double bz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(ax, bx), __dmul_rn(ay, by)), __dmul_rn(az, bz));
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

// ----------------------------------------------------- TMA / mbarrier PTX
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  }
}
// 1-D TMA bulk copy global -> shared, completing on `bar` (16-byte aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------- recomputed HG kernel blocks
// Clusters with cl_mode 0 (volume members, |g| <= 0.95: the aggregate's fp32
// HG path) store no W block; W[r, j] = num(g_r) hg3(r, j) / phat_ind[j] is
// recomputed from the row data (graph.cuh): anchor a_r and g_r (rows[4q+2]),
// phase direction d_j and 1 - |d_j|^2 (rows[4q+3]), 1/phat_ind[j]
// (rows[4q+1].w).  hg3 = (|d - g a|^2 + 1 - |d|^2)^-3/2, the aggregate's
// hg_pdf32 without the g^2 (1 - |a|^2) term (~1e-16 for the unit anchors).
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float hg3(const float4 ha, const float4 dc) {
  const float ux = fmaf(-ha.w, ha.x, dc.x), uy = fmaf(-ha.w, ha.y, dc.y),
              uz = fmaf(-ha.w, ha.z, dc.z);
  const float r = rsqrt_ftz(fmaf(ux, ux, fmaf(uy, uy, fmaf(uz, uz, dc.w))));
  return r * r * r;
}
// W[r, j] exactly as the aggregate's fp32 path evaluates it:
// (num_r * hg3) * (1 / phat_ind[j])
__device__ __forceinline__ float w_recomputed(const float4* __restrict__ rows, int64_t qr,
                                              int64_t qj) {
  const float4 ha = rows[4 * qr + 2];
  return (hg_num_f32(ha.w) * hg3(ha, rows[4 * qj + 3])) * rows[4 * qj + 1].w;
}

// One fixed-point iteration t (solve.py:78-83) over TMA-staged chunks.
//
// A persistent CTA per SM walks its chunks (see graph.cuh) with a producer
// warp and kConsumers consumer warps:
//  - the producer streams each chunk's kernel blocks, static row data
//    {a, b, par}, its slice of I and (t > 0) of the previous W*I into a
//    shared-memory stage with cp.async.bulk, n_stages chunks ahead; a stage
//    is refilled once every cluster of its chunk has been consumed;
//  - consumer warps pull clusters one at a time from a CTA-wide counter (in
//    chunk order, so a warp never waits on a slower warp), wait on the
//    chunk's mbarrier the first time they touch it, and for cluster k
//    accumulate (W I)[r] from shared memory (lane = row), then propagate the
//    row into its continuation parent, I_out[par] = a * acc + b, scattered
//    to HBM, with the residual maxima of solve.py:54-61.  The old I[par] is
//    recomputed from the previous W*I (same arithmetic as when it was stored)
//    instead of gathered.
#ifndef VPG_SOLVE_UNROLL1
#define VPG_SOLVE_UNROLL1 4  // column loop, one row per lane
#endif
#ifndef VPG_SOLVE_UNROLL2
#define VPG_SOLVE_UNROLL2 2  // column loop, two rows per lane
#endif
constexpr int kSolveUnroll1 = VPG_SOLVE_UNROLL1, kSolveUnroll2 = VPG_SOLVE_UNROLL2;
#ifndef VPG_SOLVE_CONSUMERS
#define VPG_SOLVE_CONSUMERS 24
#endif
constexpr int kConsumers = VPG_SOLVE_CONSUMERS;
constexpr int kMaxStages = 4;  // the stage count is chosen per graph (graph.cuh)

// Residual, tol break and 3-growth divergence of iteration t (solve.py:80-94),
// decided on the device so the loop never waits on the host.
__device__ void control_step(int t, double tol, const uint32_t* __restrict__ red,
                             const float* __restrict__ term_max, double* __restrict__ resid,
                             int32_t* __restrict__ ctl) {
  if (ctl[1]) return;
  // red was filled by atomics from every CTA: read it past L1
  const uint32_t* vred = red;
  double worst = 0.0;
  for (int c = 0; c < 3; ++c) {
    // maxima of non-negative values as float bits: above +inf means NaN,
    // and a NaN channel never wins Python's max(worst, q) in the reference
    const uint32_t db = __ldcg(vred + t * 8 + c), sb = __ldcg(vred + t * 8 + 3 + c);
    if (db > 0x7F800000u || sb > 0x7F800000u) continue;
    const double delta = double(__uint_as_float(db));
    double scale = double(fmaxf(__uint_as_float(sb), term_max[c]));
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

// The last CTA of iteration t to finish (counter red[t*8+7]) runs the control
// step: no separate control launch between iterations.
__device__ __forceinline__ void finish_iteration(int t, double tol, uint32_t* __restrict__ red,
                                                 const float* __restrict__ term_max,
                                                 double* __restrict__ resid,
                                                 int32_t* __restrict__ ctl) {
  __threadfence();
  const unsigned prev = atomicAdd(&red[t * 8 + 7], 1u);
  if (prev == gridDim.x - 1) {
    __threadfence();
    control_step(t, tol, red, term_max, resid, ctl);
  }
}

__global__ void __launch_bounds__((kConsumers + 1) * 32, 1)
k_solve_iter(const int4* __restrict__ desc, const int4* __restrict__ meta,
             const int64_t* __restrict__ n_chunks_p, int n_stages, int stage_floats,
             const float* __restrict__ wt, const int64_t* __restrict__ w_off,
             const float4* __restrict__ rows,
             const float4* __restrict__ i_in, float4* __restrict__ i_out,
             const float4* __restrict__ acc_prev, float4* __restrict__ acc_out,
             const float4* __restrict__ i0, int t, uint32_t* __restrict__ red,
             int32_t* __restrict__ ctl, int fused, double tol,
             const float* __restrict__ term_max, double* __restrict__ resid) {
  if (ctl[1]) return;  // converged or diverged earlier (every CTA sees the same)
  const int64_t n_chunks = *n_chunks_p;
  if (int64_t(blockIdx.x) >= n_chunks) {
    if (fused && threadIdx.x == 0) finish_iteration(t, tol, red, term_max, resid, ctl);
    return;
  }
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);             // n_stages (<= 4) barriers
  int* done = reinterpret_cast<int*>(smem + 64);                  // n_stages counters
  int* next_item = reinterpret_cast<int*>(smem + 96);
  int* issued = reinterpret_cast<int*>(smem + 104);               // n_stages chunk ids
  float* stage0 = reinterpret_cast<float*>(smem + 128);
  __shared__ uint32_t blk[kConsumers][6];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    for (int st = 0; st < n_stages; ++st) {
      mbar_init(&full[st], 1);
      done[st] = 0;
      issued[st] = -1;
    }
    *next_item = 0;
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t G = gridDim.x;

  if (wid == kConsumers) {
    // ------------------------------------------------------------ producer
    // The warp loads the descriptors of its next 32 chunks at once (one
    // 32-byte load per lane), so no dependent metadata load sits between
    // two refills; lane 0 issues the copies.
    __shared__ int prev_nk[kMaxStages];  // cluster count of the chunk last issued per stage
    for (int64_t i0c = 0;; i0c += 32) {
      const int64_t cl = blockIdx.x + (i0c + lane) * G;
      int4 d0 = make_int4(0, 0, 0, 0), d1 = d0;
      if (cl < n_chunks) {
        d0 = desc[2 * cl];
        d1 = desc[2 * cl + 1];
      }
      bool finished = false;
      for (int j = 0; j < 32; ++j) {
        const int64_t i = i0c + j;
        if (blockIdx.x + i * G >= n_chunks) {
          finished = true;
          break;
        }
        const int k0 = __shfl_sync(0xFFFFFFFFu, d0.x, j);
        const int nk = __shfl_sync(0xFFFFFFFFu, d0.y, j);
        const int q0 = __shfl_sync(0xFFFFFFFFu, d0.z, j);
        const int R = __shfl_sync(0xFFFFFFFFu, d0.w, j);
        const int wc = __shfl_sync(0xFFFFFFFFu, d1.x, j);
        const int st = int(i % n_stages);
        uint64_t* bar = &full[st];
        float* buf = stage0 + st * int64_t(stage_floats);
        if (lane == 0) {
          if (i >= n_stages) {
            // the stage's previous chunk must be fully consumed
            while (*reinterpret_cast<volatile int*>(&done[st]) < prev_nk[st]) __nanosleep(32);
            done[st] = 0;
            fence_proxy_async();  // consumers' generic reads before the async refill
          }
          // the stage's previous phase has completed (its chunk was consumed), so
          // a consumer that sees issued == i waits on this chunk's phase
          *reinterpret_cast<volatile int*>(&issued[st]) = int(i);
          if (nk == 0) {
            mbar_arrive(bar);
          } else {
            const uint32_t mb = uint32_t(nk) * 16u, wb = uint32_t(wc) * 4u,
                           rb = uint32_t(R) * 64u, ib = uint32_t(R) * 16u;
            mbar_expect_tx(bar, mb + wb + rb + ib + (t > 0 ? ib : 0u));
            bulk_g2s(buf, meta + k0, mb, bar);
            float* p = buf + 4 * nk + wc;
            bulk_g2s(p, rows + 4 * int64_t(q0), rb, bar);
            p += 16 * R;
            bulk_g2s(p, i_in + q0, ib, bar);
            if (t > 0) bulk_g2s(p + 4 * R, acc_prev + q0, ib, bar);
          }
          prev_nk[st] = nk;
        }
        if (wc > 0) {
          // stored W blocks (Lambertian / high-g clusters), one copy per
          // cluster issued by the lanes in parallel after lane 0 has claimed
          // the stage and announced the chunk's bytes
          __syncwarp();
          fence_proxy_async();
          for (int kk = lane; kk < nk; kk += 32) {
            const int4 mk = meta[k0 + kk];
            if (mk.w) {
              const int64_t sz = mk.z;
              bulk_g2s(buf + 4 * nk + mk.y, wt + w_off[k0 + kk],
                       uint32_t(((sz * sz + 3) & ~int64_t(3)) * 4), bar);
            }
          }
        }
      }
      if (finished) break;
    }
  } else {
    // ----------------------------------------------------------- consumers
    uint32_t dmax[3] = {0u, 0u, 0u}, smax[3] = {0u, 0u, 0u};  // float bits (see epilogue)
    int64_t ci = 0, cbase = 0, waited = -1;  // current chunk (local index), its first item
    int nk = 0, R = 0, wc = 0, cq0 = 0;      // of chunk ci
    {
      const int64_t c = blockIdx.x;
      if (c < n_chunks) {
        const int4 d0 = desc[2 * c], d1 = desc[2 * c + 1];
        nk = d0.y;
        cq0 = d0.z;
        R = d0.w;
        wc = d1.x;
      }
    }
    for (;;) {
      int x = 0;
      if (lane == 0) x = atomicAdd(next_item, 1);
      x = __shfl_sync(0xFFFFFFFFu, x, 0);
      // advance to the chunk holding item x (immutable descriptors: no race
      // with the producer reusing a stage)
      bool finished = false;
      while (true) {
        const int64_t c = blockIdx.x + ci * G;
        if (c >= n_chunks) {
          finished = true;
          break;
        }
        if (x < cbase + nk) break;
        cbase += nk;
        ++ci;
        const int64_t c2 = blockIdx.x + ci * G;
        if (c2 < n_chunks) {
          const int4 d0 = desc[2 * c2], d1 = desc[2 * c2 + 1];
          nk = d0.y;
          cq0 = d0.z;
          R = d0.w;
          wc = d1.x;
        }
      }
      if (finished) break;
      const int st = int(ci % n_stages);
      if (waited != ci) {
        // never wait on a phase parity two uses ahead: first see the chunk issued
        while (*reinterpret_cast<volatile int*>(&issued[st]) != int(ci)) __nanosleep(32);
        mbar_wait(&full[st], uint32_t((ci / n_stages) & 1));
        waited = ci;
      }
      const float* buf = stage0 + st * int64_t(stage_floats);
      const int4* smeta = reinterpret_cast<const int4*>(buf);
      const int4 mk = smeta[x - cbase];
      const float* wbase = buf + 4 * nk;
      const float4* srow = reinterpret_cast<const float4*>(wbase + wc);
      const float4* sin = reinterpret_cast<const float4*>(wbase + wc + 16 * int64_t(R));
      const float4* sprev = reinterpret_cast<const float4*>(wbase + wc + 20 * int64_t(R));
      // row rr (position in its cluster, rows from crow / q0) with its
      // W*I: acc_out, the terminal carry, the scatter into the parent and
      // the residual maxima.  The maxima are kept as IEEE bit patterns of
      // non-negative values: an integer max orders NaN above +inf, so a NaN
      // propagates like numpy's max (solve.py:54-61).
      auto epilogue = [&](const float4* crow, int rl, int64_t q0, int rr, float ax, float ay,
                          float az) {
        const int64_t q = q0 + rr;
        acc_out[q] = make_float4(ax, ay, az, 0.f);
        const float4 A = crow[4 * rr], B = crow[4 * rr + 1];
        const int32_t link = __float_as_int(A.w);
        // a terminal row's I stays i_pt: written into both I buffers by the
        // first two iterations, never touched again
        if (t < 2 && link_terminal(link)) i_out[q] = i0[q];
        const int32_t p = link_parent(link);
        if (p < 0) return;
        const float nx = fmaf(A.x, ax, B.x), ny = fmaf(A.y, ay, B.y), nz = fmaf(A.z, az, B.z);
        float4 old;
        if (t == 0) {
          old = i0[p];
        } else {
          const float4 pa = sprev[rl + rr];
          old = make_float4(fmaf(A.x, pa.x, B.x), fmaf(A.y, pa.y, B.y), fmaf(A.z, pa.z, B.z), 0.f);
        }
        i_out[p] = make_float4(nx, ny, nz, 0.f);
        dmax[0] = max(dmax[0], __float_as_uint(fabsf(nx - old.x)));
        dmax[1] = max(dmax[1], __float_as_uint(fabsf(ny - old.y)));
        dmax[2] = max(dmax[2], __float_as_uint(fabsf(nz - old.z)));
        smax[0] = max(smax[0], __float_as_uint(fabsf(nx)));
        smax[1] = max(smax[1], __float_as_uint(fabsf(ny)));
        smax[2] = max(smax[2], __float_as_uint(fabsf(nz)));
      };
      const int items = 1;
      if (mk.w == 0) {
        // W recomputed from the row data: num_r hg3(r, j) / phat_ind[j], the
        // aggregate's fp32 HG terms (the products grouped per row and per
        // column instead of per pair).  Rows go to lanes in passes chosen to keep
        // the lanes busy: 64 rows as two per lane, 17..32 rows one per lane,
        // and up to 16 rows as column slices -- P = 32 / pow2(rows) lanes per
        // row, each summing every P-th column, combined by xor shuffles.
        const int rl = mk.x;
        const int s = mk.z;
        VPG_CHECK(rl >= 0 && s >= 1 && rl + s <= R);  // the cluster's rows are staged
        const int64_t q0 = int64_t(cq0) + rl;
        const float4* crow = srow + 4 * rl;
        const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (s == 1) {
          // a lone record: W = phat * (1 / phat), evaluated exactly as the
          // aggregate did, so that at K = 1 the fixed point (the PT
          // estimate, reached at once) shows no fp32 noise growth
          if (lane == 0) {
            const float4 ha = crow[2], ij = sin[rl];
            const float wv = (hg_num_f32(ha.w) * hg3(ha, crow[3])) * crow[1].w;
            epilogue(crow, rl, q0, 0, wv * ij.x, wv * ij.y, wv * ij.z);
          }
          __syncwarp();
          if (lane == 0) atomicAdd(&done[st], 1);
          continue;
        }
        // W[r, j] I_j = num_r hg3(r, j) (1/phat_ind[j] I_j): the column
        // factor is applied to the staged I once per column (in place: only
        // this cluster reads these rows of I), num_r once per row
        {
          float4* icol = const_cast<float4*>(sin) + rl;
          for (int j = lane; j < s; j += 32) {
            const float iw = crow[4 * j + 1].w;
            float4 v = icol[j];
            v.x *= iw;
            v.y *= iw;
            v.z *= iw;
            icol[j] = v;
          }
          __syncwarp();
        }
        // one row (anchor ha) over columns j0, j0 + dj, ... < s, times num n
        auto one_row = [&](const float4 ha, float n, int j0, int dj) {
          float3 acc = make_float3(0.f, 0.f, 0.f);
#pragma unroll kSolveUnroll1
          for (int j = j0; j < s; j += dj) {
            const float4 dc = crow[4 * j + 3];
            const float4 ij = sin[rl + j];
            const float h = hg3(ha, dc);
            acc.x = fmaf(h, ij.x, acc.x);
            acc.y = fmaf(h, ij.y, acc.y);
            acc.z = fmaf(h, ij.z, acc.z);
          }
          return make_float3(acc.x * n, acc.y * n, acc.z * n);
        };
        int rc = 0;
        while (rc < s) {
          const int rem = s - rc;
          if (rem > 48) {
            // two rows per lane, the column data loaded once for both
            const int r0 = rc + lane, r1 = rc + lane + 32;
            const float4 ha0 = crow[4 * r0 + 2];
            const float4 ha1 = r1 < s ? crow[4 * r1 + 2] : z4;
            const float n0 = hg_num_f32(ha0.w), n1 = hg_num_f32(ha1.w);
            float3 acc0 = make_float3(0.f, 0.f, 0.f), acc1 = acc0;
#pragma unroll kSolveUnroll2
            for (int j = 0; j < s; ++j) {
              const float4 dc = crow[4 * j + 3];
              const float4 ij = sin[rl + j];
              const float h0 = hg3(ha0, dc), h1 = hg3(ha1, dc);
              acc0.x = fmaf(h0, ij.x, acc0.x);
              acc0.y = fmaf(h0, ij.y, acc0.y);
              acc0.z = fmaf(h0, ij.z, acc0.z);
              acc1.x = fmaf(h1, ij.x, acc1.x);
              acc1.y = fmaf(h1, ij.y, acc1.y);
              acc1.z = fmaf(h1, ij.z, acc1.z);
            }
            epilogue(crow, rl, q0, r0, acc0.x * n0, acc0.y * n0, acc0.z * n0);
            if (r1 < s) epilogue(crow, rl, q0, r1, acc1.x * n1, acc1.y * n1, acc1.z * n1);
            rc += 64;
          } else if (rem > 16) {
            // one row per lane (32 rows; 17..32 at the end)
            const int r = rc + lane;
            const bool on = lane < rem;
            const float4 ha = on ? crow[4 * r + 2] : z4;
            const float3 acc = one_row(ha, hg_num_f32(ha.w), 0, 1);
            if (on) epilogue(crow, rl, q0, r, acc.x, acc.y, acc.z);
            rc += rem > 32 ? 32 : rem;
          } else {
            // <= 16 rows: P lanes per row on every P-th column
            const int w2 = rem <= 1 ? 1 : (rem <= 2 ? 2 : (rem <= 4 ? 4 : (rem <= 8 ? 8 : 16)));
            const int P = 32 / w2;
            const int rr = lane & (w2 - 1), h = lane / w2;
            const bool on = rr < rem;
            const int r = rc + rr;
            const float4 ha = on ? crow[4 * r + 2] : z4;
            float3 acc = on ? one_row(ha, 1.f, h, P) : make_float3(0.f, 0.f, 0.f);
            for (int off = w2; off < 32; off <<= 1) {
              acc.x += __shfl_xor_sync(0xFFFFFFFFu, acc.x, off);
              acc.y += __shfl_xor_sync(0xFFFFFFFFu, acc.y, off);
              acc.z += __shfl_xor_sync(0xFFFFFFFFu, acc.z, off);
            }
            const float n = hg_num_f32(ha.w);
            if (on && h == 0) epilogue(crow, rl, q0, r, acc.x * n, acc.y * n, acc.z * n);
            rc += rem;
          }
        }
      } else {
        // stored W block (Lambertian / |g| > 0.95 clusters), lane = row
        const int rl = mk.x;
        const int s = mk.z;
        VPG_CHECK(rl >= 0 && rl + s <= R && mk.y >= 0 && int64_t(mk.y) + int64_t(s) * s <= wc);
        const int64_t q0 = int64_t(cq0) + rl;
        const float* w = wbase + mk.y;
        const float4* crow = srow + 4 * rl;
        for (int rc = 0; rc < s; rc += 64) {
          const int r0 = rc + lane, r1 = rc + lane + 32;
          float3 acc0 = make_float3(0.f, 0.f, 0.f), acc1 = acc0;
          if (s - rc <= 32) {
            const float* colr = w + r0;
#pragma unroll 4
            for (int j = 0; j < s; ++j) {
              const float4 ij = sin[rl + j];
              const float w0v = r0 < s ? colr[j * s] : 0.f;
              acc0.x = fmaf(w0v, ij.x, acc0.x);
              acc0.y = fmaf(w0v, ij.y, acc0.y);
              acc0.z = fmaf(w0v, ij.z, acc0.z);
            }
          } else {
#pragma unroll 4
            for (int j = 0; j < s; ++j) {
              const float4 ij = sin[rl + j];
              const float* col = w + j * s;
              const float w0v = r0 < s ? col[r0] : 0.f;
              const float w1v = r1 < s ? col[r1] : 0.f;
              acc0.x = fmaf(w0v, ij.x, acc0.x);
              acc0.y = fmaf(w0v, ij.y, acc0.y);
              acc0.z = fmaf(w0v, ij.z, acc0.z);
              acc1.x = fmaf(w1v, ij.x, acc1.x);
              acc1.y = fmaf(w1v, ij.y, acc1.y);
              acc1.z = fmaf(w1v, ij.z, acc1.z);
            }
          }
          if (r0 < s) epilogue(crow, rl, q0, r0, acc0.x, acc0.y, acc0.z);
          if (r1 < s) epilogue(crow, rl, q0, r1, acc1.x, acc1.y, acc1.z);
        }
      }
      __syncwarp();
      if (lane == 0) atomicAdd(&done[st], items);
    }
    uint32_t v[6] = {dmax[0], dmax[1], dmax[2], smax[0], smax[1], smax[2]};
#pragma unroll
    for (int q = 0; q < 6; ++q)
      for (int off = 16; off; off >>= 1) v[q] = max(v[q], __shfl_xor_sync(0xFFFFFFFFu, v[q], off));
    if (lane == 0)
      for (int q = 0; q < 6; ++q) blk[wid][q] = v[q];
  }
  __syncthreads();
  if (tid < 6) {
    uint32_t x = 0u;
    for (int w2 = 0; w2 < kConsumers; ++w2) x = max(x, blk[w2][tid]);
    if (x) atomicMax(&red[t * 8 + tid], x);
  }
  if (fused) {
    __syncthreads();  // this CTA's maxima are in
    if (tid == 0) finish_iteration(t, tol, red, term_max, resid, ctl);
  }
}

// W * v per cluster from global memory (aggregate_indirect on an arbitrary
// vector; not on the solve path).  Warp per cluster.
constexpr int kItWarps = 8;
__global__ void __launch_bounds__(kItWarps * 32)
k_apply_w(const int32_t* __restrict__ cl_off, const int64_t* __restrict__ w_off, int64_t m,
          const float* __restrict__ wt, const uint8_t* __restrict__ cl_mode,
          const float4* __restrict__ rows, const float4* __restrict__ v_in,
          float4* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = int64_t(gridDim.x) * kItWarps;
  for (int64_t k = int64_t(blockIdx.x) * kItWarps + (threadIdx.x >> 5); k < m; k += nwarps) {
    const int32_t q0 = cl_off[k];
    const int s = cl_off[k + 1] - q0;
    const float* w = wt + w_off[k];
    const bool stored = cl_mode[k] != 0;
    for (int r = lane; r < s; r += 32) {
      float3 acc = make_float3(0.f, 0.f, 0.f);
      for (int j = 0; j < s; ++j) {
        const float4 vj = v_in[q0 + j];
        const float wv = stored ? w[int64_t(j) * s + r] : w_recomputed(rows, q0 + r, q0 + j);
        acc.x = fmaf(wv, vj.x, acc.x);
        acc.y = fmaf(wv, vj.y, acc.y);
        acc.z = fmaf(wv, vj.z, acc.z);
      }
      out[q0 + r] = make_float4(acc.x, acc.y, acc.z, 0.f);
    }
  }
}

// Residual bookkeeping for iteration t (solve.py:54-61,80-94).
// ctl = {performed, stop, grow, diverged}
__global__ void k_control(int t, double tol, const uint32_t* __restrict__ red,
                          const float* __restrict__ term_max, double* __restrict__ resid,
                          int32_t* __restrict__ ctl) {
  if (threadIdx.x == 0) control_step(t, tol, red, term_max, resid, ctl);
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

__global__ void k_row_sizes(const int32_t* __restrict__ cluster_id,
                            const int32_t* __restrict__ internal_of,
                            const int32_t* __restrict__ cl_size, int64_t n, int64_t* __restrict__ sz) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r <= n;
       r += int64_t(gridDim.x) * blockDim.x) {
    if (r == n) { sz[r] = 0; continue; }
    sz[r] = cl_size[internal_of[cluster_id[r]]];
  }
}

// Clusters in the reference's numbering: sizes, member lists, centers.
__global__ void k_ref_sizes(const int32_t* __restrict__ internal_of,
                            const int32_t* __restrict__ cl_size, int64_t m, int64_t* __restrict__ sz) {
  for (int64_t rr = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; rr <= m;
       rr += int64_t(gridDim.x) * blockDim.x)
    sz[rr] = rr < m ? cl_size[internal_of[rr]] : 0;
}

__global__ void k_ref_members(const int32_t* __restrict__ internal_of,
                              const int32_t* __restrict__ cl_off, const int32_t* __restrict__ cl_size,
                              const int32_t* __restrict__ cl_center, const int32_t* __restrict__ perm,
                              const int64_t* __restrict__ off, int64_t m, int64_t* __restrict__ members,
                              int64_t* __restrict__ centers) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t rr = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; rr < m; rr += warps) {
    const int32_t k = internal_of[rr];
    const int32_t q0 = cl_off[k], sz = cl_size[k];
    for (int32_t t = lane; t < sz; t += 32) members[off[rr] + t] = perm[q0 + t];
    if (lane == 0) centers[rr] = cl_center[k];
  }
}

// CSR rows of W in record order (graph.py:167): warp per row.
__global__ void k_export_csr(const int32_t* __restrict__ cluster_id,
                             const int32_t* __restrict__ internal_of, const int32_t* __restrict__ clpos,
                             const int32_t* __restrict__ cl_off, const int32_t* __restrict__ cl_size,
                             const int64_t* __restrict__ w_off, const int32_t* __restrict__ perm,
                             const float* __restrict__ wt, const uint8_t* __restrict__ cl_mode,
                             const float4* __restrict__ rows, const int64_t* __restrict__ indptr,
                             int64_t n, int64_t* __restrict__ indices, double* __restrict__ data) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; r < n; r += nwarps) {
    const int32_t k = internal_of[cluster_id[r]];
    const int32_t q0 = cl_off[k];
    const int s = cl_size[k];
    const int rl = clpos[r] - q0;
    const int64_t base = indptr[r];
    const bool stored = cl_mode[k] != 0;
    for (int j = lane; j < s; j += 32) {
      indices[base + j] = perm[q0 + j];
      data[base + j] = double(stored ? wt[w_off[k] + int64_t(j) * s + rl]
                                     : w_recomputed(rows, q0 + rl, q0 + j));
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

// ------------------------------------------------------------------ solve
// solve() = solve_begin + iterations x (solve_step + solve_control) + solve_end.
// A shard-local graph runs the same pieces with the halo exchange and the
// residual all-reduce between solve_step and solve_control (pathgraph/sharded.py).
namespace {
struct SolveLaunch {
  int stage_floats = 0;
  size_t smem = 0;
  int grid = 0;
};

SolveLaunch solve_launch(const vpg_graph* g) {
  // stage = one chunk (g->chunk_floats) plus the largest cluster's blocks + rows
  SolveLaunch L;
  const int smax = std::max(1, g->max_cluster);
  L.stage_floats = g->chunk_floats + ((smax * smax + 3) & ~3) + kRowFloats * smax + 4;
  L.smem = 128 + size_t(g->n_stages) * L.stage_floats * sizeof(float);
  VPG_REQUIRE(L.smem <= kSolveSmem, VPG_ELIMIT, "clusters too large for the staged solve");
  ensure_dynamic_smem(reinterpret_cast<const void*>(k_solve_iter), L.smem);
  L.grid = sm_count();  // persistent; CTAs past the (device-side) chunk count exit
  return L;
}
}  // namespace

void solve_begin(vpg_graph* g, const vpg_records& rec, int32_t iterations, double tol,
                 cudaStream_t s) {
  VPG_REQUIRE(iterations >= 0, VPG_EINVAL, "iterations must be >= 0");
  const int64_t n = g->n;
  if (g->red_cap < iterations + 1) {
    g->red.alloc(size_t(iterations + 1) * 8, s);
    g->resid.alloc(size_t(iterations + 1), s);
    g->red_cap = iterations + 1;
  }
  if (!g->ctl.get()) g->ctl.alloc(4, s);
  g->tol = tol;
  g->iterations = iterations;
  g->performed = -1;
  VPG_CUDA(cudaMemsetAsync(g->red.get(), 0, g->red.bytes(), s));
  VPG_CUDA(cudaMemsetAsync(g->ctl.get(), 0, 4 * sizeof(int32_t), s));
  const int block = 256;
  // the iterations read I_0 from i0 and carry the terminal rows themselves
  // (rows flagged in rows[].w); only a solve of 0 iterations reads ibuf[0]
  if (n > 0 && iterations == 0) {
    VPG_LAUNCH(k_fill_f4, grid_for(n, block), block, 0, s, g->ibuf[0].get(), g->i0.get(), n);
    VPG_LAUNCH(k_own_indirect, grid_for(n, block), block, 0, s, rec, g->perm.get(), n,
               g->acc[0].get());
  }
}

namespace {
void launch_iteration(vpg_graph* g, int32_t t, bool fused, cudaStream_t s) {
  VPG_REQUIRE(t >= 0 && t < g->iterations, VPG_EINVAL, "iteration index out of range");
  if (g->n == 0) return;
  const SolveLaunch L = solve_launch(g);
  VPG_LAUNCH(k_solve_iter, L.grid, (kConsumers + 1) * 32, L.smem, s, g->chunk_desc.get(),
             g->cl_meta.get(), g->n_chunks_dev.get(), g->n_stages, L.stage_floats, g->wt.get(),
             g->w_off.get(), g->rows.get(), t == 0 ? g->i0.get() : g->ibuf[t & 1].get(),
             g->ibuf[(t + 1) & 1].get(), g->acc[t & 1].get(),
             g->acc[(t + 1) & 1].get(), g->i0.get(), t, g->red.get(), g->ctl.get(),
             fused ? 1 : 0, g->tol, g->term_max.get(), g->resid.get());
}
}  // namespace

// one iteration without its control step (a shard runs the halo exchange and
// the residual all-reduce in between, then solve_control)
void solve_step(vpg_graph* g, int32_t t, cudaStream_t s) { launch_iteration(g, t, false, s); }

void solve_control(vpg_graph* g, int32_t t, cudaStream_t s) {
  VPG_REQUIRE(t >= 0 && t < g->iterations, VPG_EINVAL, "iteration index out of range");
  VPG_LAUNCH(k_control, 1, 32, 0, s, t, g->tol, g->red.get(), g->term_max.get(), g->resid.get(),
             g->ctl.get());
}

void solve_end(vpg_graph* g, double* residuals, int32_t* performed, bool empty, cudaStream_t s) {
  const int32_t iterations = g->iterations;
  int32_t ctl_h[4] = {0, 0, 0, 0};
  if (!empty && iterations > 0) {
    VPG_CUDA(cudaMemcpyAsync(ctl_h, g->ctl.get(), sizeof(ctl_h), cudaMemcpyDeviceToHost, s));
    VPG_CUDA(cudaMemcpyAsync(residuals, g->resid.get(), sizeof(double) * iterations,
                             cudaMemcpyDeviceToHost, s));
    count_transfer(0, sizeof(ctl_h) + sizeof(double) * iterations);
  } else if (iterations > 0) {
    // an empty graph: every residual is 0/1e-12 = 0 and the tol test stops at once
    for (int t = 0; t < iterations; ++t) residuals[t] = 0.0;
    ctl_h[0] = g->tol > 0.0 ? 1 : iterations;
  }
  VPG_CUDA(cudaStreamSynchronize(s));
  g->performed = ctl_h[0];
  *performed = ctl_h[0];
  if (ctl_h[3]) throw Error(VPG_EDIVERGED, "fixed-point residuals grew over 3 consecutive iterations");
}

void solve(vpg_graph* g, const vpg_records& rec, int32_t iterations, double tol,
           double* residuals, int32_t* performed, cudaStream_t s) {
  solve_begin(g, rec, iterations, tol, s);
  const int64_t n = g->n;
  for (int t = 0; t < iterations && n > 0; ++t) {
    launch_iteration(g, t, true, s);  // control step in the iteration's last CTA
  }
  solve_end(g, residuals, performed, n == 0, s);
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
  VPG_LAUNCH(k_apply_w, iterate_grid(g->m), kItWarps * 32, 0, s, g->cl_off.get(),
             g->w_off.get(), g->m, g->wt.get(), g->cl_mode.get(), g->rows.get(), vin.get(),
             vout.get());
  VPG_LAUNCH(k_scatter_rec3, grid_for(n, block), block, 0, s, vout.get(), g->clpos.get(),
             rec.coeff, n, out);
}

void propagate(const vpg_records& rec, const double* lbar, double* out, int linear,
               cudaStream_t s) {
  if (rec.n == 0) return;
  VPG_LAUNCH(k_propagate, grid_for(rec.n, 256), 256, 0, s, rec, lbar, linear, out);
}

namespace {
// record -> reference cluster number, warp per cluster (exports only)
__global__ void k_cluster_ids(const int32_t* __restrict__ cl_off, const int32_t* __restrict__ cl_size,
                              const int32_t* __restrict__ ref_of, const int32_t* __restrict__ perm,
                              int64_t m, int32_t* __restrict__ cluster_id) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t k = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; k < m; k += warps) {
    const int32_t q0 = cl_off[k], sz = cl_size[k], ref = ref_of[k];
    for (int32_t t = lane; t < sz; t += 32) cluster_id[perm[q0 + t]] = ref;
  }
}
}  // namespace

void ensure_cluster_ids(const vpg_graph* g, cudaStream_t s) {
  if (g->cluster_id_ready) return;
  if (g->n > 0)
    VPG_LAUNCH(k_cluster_ids, grid_for(g->m * 32, 256), 256, 0, s, g->cl_off.get(),
               g->cl_size.get(), g->ref_of.get(), g->perm.get(), g->m,
               const_cast<int32_t*>(g->cluster_id.get()));
  g->cluster_id_ready = true;
}

void export_clusters(const vpg_graph* g, int64_t* cluster_id, int64_t* cl_off, int64_t* members,
                     int64_t* centers, cudaStream_t s) {
  ensure_cluster_ids(g, s);
  const int64_t n = g->n, m = g->m;
  const int block = 256;
  if (cluster_id && n) {
    DBuf<int64_t> tmp(n, s);
    VPG_LAUNCH(k_i32_to_i64, grid_for(n, block), block, 0, s, g->cluster_id.get(), n, tmp.get());
    VPG_CUDA(cudaMemcpyAsync(cluster_id, tmp.get(), n * 8, cudaMemcpyDeviceToHost, s));
    VPG_CUDA(cudaStreamSynchronize(s));
  }
  if (!(cl_off || members || centers)) return;
  DBuf<int64_t> sz(m + 1, s), off(m + 1, s), mem(n + 1, s), cen(m + 1, s);
  VPG_LAUNCH(k_ref_sizes, grid_for(m + 1, block), block, 0, s, g->internal_of.get(),
             g->cl_size.get(), m, sz.get());
  size_t bytes = 0;
  VPG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, sz.get(), off.get(), int(m + 1), s));
  {
    DBuf<char> t(bytes, s);
    VPG_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), bytes, sz.get(), off.get(), int(m + 1), s));
    count_launch(1);
  }
  VPG_LAUNCH(k_ref_members, grid_for(m * 32, block), block, 0, s, g->internal_of.get(),
             g->cl_off.get(), g->cl_size.get(), g->cl_center.get(), g->perm.get(), off.get(), m,
             mem.get(), cen.get());
  if (cl_off) VPG_CUDA(cudaMemcpyAsync(cl_off, off.get(), (m + 1) * 8, cudaMemcpyDeviceToHost, s));
  if (members && n) VPG_CUDA(cudaMemcpyAsync(members, mem.get(), n * 8, cudaMemcpyDeviceToHost, s));
  if (centers && m) VPG_CUDA(cudaMemcpyAsync(centers, cen.get(), m * 8, cudaMemcpyDeviceToHost, s));
  VPG_CUDA(cudaStreamSynchronize(s));
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
  ensure_cluster_ids(g, s);
  const int64_t n = g->n;
  if (n == 0) {
    if (indptr) indptr[0] = 0;
    return;
  }
  const int block = 256;
  if (indptr || indices || data) {
    DBuf<int64_t> sz(n + 1, s), ip(n + 1, s);
    VPG_LAUNCH(k_row_sizes, grid_for(n + 1, block), block, 0, s, g->cluster_id.get(),
               g->internal_of.get(), g->cl_size.get(), n, sz.get());
    size_t bytes = 0;
    VPG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, sz.get(), ip.get(), int(n + 1), s));
    {
      DBuf<char> t(bytes, s);
      VPG_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), bytes, sz.get(), ip.get(), int(n + 1), s));
      count_launch(1);
    }
    if (indptr) VPG_CUDA(cudaMemcpyAsync(indptr, ip.get(), (n + 1) * 8, cudaMemcpyDeviceToHost, s));
    if (indices || data) {
      g->sync_totals();
      DBuf<int64_t> ind(size_t(g->nnz) + 1, s);
      DBuf<double> dat(size_t(g->nnz) + 1, s);
      VPG_LAUNCH(k_export_csr, grid_for(n * 32, block), block, 0, s, g->cluster_id.get(),
                 g->internal_of.get(), g->clpos.get(), g->cl_off.get(), g->cl_size.get(),
                 g->w_off.get(), g->perm.get(), g->wt.get(), g->cl_mode.get(), g->rows.get(),
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

void splat_arrays(const vpg_paths& P, const double* coeff, const int32_t* clpos, const float4* acc,
                  const float4* dbar, int64_t npix, int spp, int mode, double* image,
                  cudaStream_t s) {
  VPG_REQUIRE(spp >= 1 && P.n == npix * spp, VPG_EINVAL, "path table size != pixels*spp");
  if (npix == 0) return;
  VPG_LAUNCH(k_splat, grid_for(npix, 128), 128, 0, s, P, coeff, clpos, acc, dbar, npix, spp, mode,
             image);
}

void splat_pt(const vpg_paths& P, int w, int h, int spp, double* image, cudaStream_t s) {
  VPG_REQUIRE(P.n == int64_t(w) * h * spp, VPG_EINVAL, "path table size != width*height*spp");
  const int64_t npix = int64_t(w) * h;
  VPG_LAUNCH(k_splat_pt, grid_for(npix, 128), 128, 0, s, P, npix, spp, image);
}

}  // namespace vpg

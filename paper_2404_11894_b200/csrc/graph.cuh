// Device-resident path graph (the native half of PathGraph, graph.py:29-53).
//
// Layout in HBM (N records, M clusters, nnz = sum of size^2):
//   perm[q]      int32   cluster-major position q -> record index; clusters are
//                        contiguous, members ascending (clustering.py:87-93)
//   clpos[r]     int32   record -> cluster-major position (inverse of perm)
//   cluster_id[r]int32   record -> cluster number (reference numbering)
//   Internally clusters are ordered [groups that needed no split, in group
//   order | split results]: the first part is packed and aggregated on the
//   device while the host runs the split loop.  ref_of[k] / internal_of[r]
//   map internal order <-> the reference's cluster numbering.
//   cl_off[k]    int32   (M+1) start of cluster k in cluster-major order
//   cl_size[k]   int32   members of cluster k
//   w_off[k]     int64   (M+1) start of cluster k's dense kernel block (blocks
//                        padded to 4 floats so every block is 16-byte aligned)
//   wt[]         float   nnz   per cluster an s x s block stored transposed:
//                        wt[w_off + j*s + r] = W[r, j] = rho_r(w_j)/phat_ind[j]
//                        (graph.py:143-148), columns implicit
//   phat[3][N]   double  phat_ind / phat_dir_phase / phat_dir_emit, cluster-major
//   Solve vectors, cluster-major (xyz = RGB):
//     rows[4q..4q+3]  64 bytes per row:
//              {a = w_cont*coeff, link}, {b = w_cont*D-bar, 1/phat_ind},
//              {HG anchor -omega_out (float), g}, {phase_dir (float), 1 - |d|^2}
//              link = (par + 1) * 2 + terminal, par = position of the
//              continuation parent (record r-1 on the same path), -1 for a
//              path's first record; terminal = no continuation child.  Row q
//              propagates into par:  I[par] = w_cont*(coeff*(W I)[q] + D-bar[q])
//              = a*acc + b.  The last two float4 are what the solve needs to
//              recompute W[r, j] = num(g_r) (|d_j - g_r a_r|^2 + 1 - |d_j|^2)^-3/2
//              / phat_ind[j] for clusters whose W block is not stored
//   cl_mode[k] uint8   1: cluster k's W block is stored in wt (Lambertian
//              members or |g| > 0.95, fp64 densities); 0: the solve recomputes
//              it in fp32 from the row data (the aggregate's fp32 HG path)
//     i0 = i_pt, dbar = D-bar, coeff (float4)
//   ibuf[2], acc[2]: double-buffered I and W*I (acc = i_bar / coeff).
//   chunk_first[c]: first cluster of solve chunk c; chunks cut the cost prefix
//     sum(pad4(s^2) + 16 s + 4) floats at multiples of chunk_floats, so one
//     chunk's cluster table, kernel blocks and row data fit a shared-memory
//     stage (TMA bulk copies).
//   chunk_desc[c]: {k0, nk, q0, R}, {wc, 0, 0, 0}: first cluster, cluster
//     count, first row, row count, staged W floats (stored blocks only) --
//     one 32-byte load.
//   cl_meta[k]: {first row - chunk's q0, staged W offset, size, cl_mode},
//     staged with the chunk so a consumer never reads cluster metadata from HBM.
#pragma once
#include <memory>
#include <vector>

#include "common.cuh"

struct vpg_graph {
  cudaStream_t stream = nullptr;
  int64_t n = 0, m = 0, nnz = 0, wt_len = 0;
  int32_t K = 0;
  vpg::DBuf<int32_t> perm, clpos, cluster_id, cl_off, cl_size, cl_center, ref_of, internal_of;
  vpg::DBuf<int64_t> w_off;
  vpg::DBuf<float> wt;
  vpg::DBuf<double> phat;
  vpg::DBuf<float4> i0, dbar, coeff, ibuf[2], acc[2];
  vpg::DBuf<float4> rows;  // 4 float4 per row (see above)
  vpg::DBuf<uint8_t> cl_mode;  // per cluster: 1 = W block stored, 0 = recomputed
  vpg::DBuf<int32_t> chunk_first;
  vpg::DBuf<int4> chunk_desc;  // 2 int4 per chunk (see above)
  vpg::DBuf<int4> cl_meta;
  vpg::DBuf<int64_t> n_chunks_dev;  // the chunk count, computed on the device
  int64_t chunk_cap = 0;            // capacity of the chunk arrays (a host-side bound)
  int32_t chunk_floats = 0, n_stages = 0;  // solve staging (finalize_chunks)
  vpg::DBuf<float> term_max;   // 3: max |i_pt| over terminal rows
  // solve state (device): red[t*8 + 0..5] float bits, ctl = {performed, stop, grow, diverged}
  vpg::DBuf<uint32_t> red;
  vpg::DBuf<double> resid;
  vpg::DBuf<int32_t> ctl;
  int32_t red_cap = 0;
  int32_t performed = -1;  // -1 = no solve yet
  // cluster_id (record -> reference cluster number) is only read by exports:
  // the build leaves it to vpg::ensure_cluster_ids on first use
  mutable bool cluster_id_ready = true;
  double tol = 0.0;        // of the solve in progress (vpg_solve_begin)
  int32_t iterations = 0;
  // shard-local graphs (vpg_graph_build_local): rows whose continuation
  // parent lives on another shard propagate into halo slots n .. n+n_halo-1
  // of the I vectors, which the caller exchanges between iterations
  int64_t n_halo = 0;
  int32_t max_cluster = 0;
  vpg_graph_info info{};
  // the records the graph was built from (borrowed; the caller keeps them alive)
  vpg_records rec{};
  // The build returns without waiting for the device: its totals arrive in
  // pinned memory (sync_totals() before reading nnz / wt_len), and pinned
  // inputs its last kernels still read are held until done_ev.
  mutable vpg::HostBuf<int64_t> tot_host;
  mutable bool tot_pending = false;
  cudaEvent_t done_ev = nullptr;
  std::vector<std::shared_ptr<void>> hold;

  void sync_totals() const {
    if (!tot_pending) return;
    cudaEventSynchronize(done_ev);
    auto* self = const_cast<vpg_graph*>(this);
    self->nnz = tot_host[0];
    self->wt_len = tot_host[1];
    self->info.nnz = nnz;
    tot_pending = false;
  }
  template <class T>
  void hold_host(std::unique_ptr<vpg::HostBuf<T>> b) {
    if (b) hold.push_back(std::shared_ptr<void>(b.release(), [](void* p) {
      delete static_cast<vpg::HostBuf<T>*>(p);
    }));
  }
  ~vpg_graph() {
    if (done_ev) {
      cudaEventSynchronize(done_ev);
      cudaEventDestroy(done_ev);
    }
    hold.clear();
  }
};

namespace vpg {
// floats of kernel blocks + row data per solve chunk (one shared-memory stage):
// chosen per graph so that n_stages stages of chunk + the largest cluster fit
// the shared memory (kSolveSmem); larger chunks keep more bytes in flight
constexpr int kChunkFloatsMax = 16384;
constexpr int kChunkFloatsMin = 2048;
constexpr size_t kSolveSmem = 226 * 1024;
// staged floats per row in a solve chunk: 16 row data + 4 I + 4 previous W*I
constexpr int kRowFloats = 24;
// row link word: (parent + 1) * 2 + terminal (parent in [-1, 2^31 - 2])
__host__ __device__ __forceinline__ int32_t row_link(int32_t parent, bool terminal) {
  return int32_t((uint32_t(parent + 1) << 1) | (terminal ? 1u : 0u));
}
__host__ __device__ __forceinline__ int32_t link_parent(int32_t link) {
  return int32_t(uint32_t(link) >> 1) - 1;
}
__host__ __device__ __forceinline__ bool link_terminal(int32_t link) { return link & 1; }
// HG normalisation (1 - g^2) / 4pi in fp32, shared by the aggregate's fp32 HG
// path and the solve's recomputed blocks (bit-identical W in both)
__host__ __device__ __forceinline__ float hg_num_f32(float g) {
  return float(1.0 / (4.0 * 3.14159265358979323846)) * fmaf(-g, g, 1.f);
}
// set row q's parent, keeping its terminal bit
__device__ __forceinline__ void set_row_parent(float4* rows, int64_t q, int32_t parent) {
  int32_t* w = reinterpret_cast<int32_t*>(rows) + 16 * q + 3;
  *w = row_link(parent, link_terminal(*w));
}
// cluster.cu: the whole build (clusters, layout, and the operator passes
// below, overlapped with the host split loop); `with_operators` = false for
// cluster_points.
void build_graph(vpg_graph* g, const vpg_records& rec, int32_t K, vpg_pcg64* rng, bool timings,
                 bool with_operators, cudaStream_t s, cudaEvent_t fields_ready = nullptr);
// aggregation.cu
size_t member_bytes();
void alloc_operator_buffers(vpg_graph* g, int64_t wt_capacity, cudaStream_t s);
// *flag (device) = 1 when some record needs a stored W block (surface, |g| > kG32)
void launch_needs_stored_w(const vpg_records& rec, int32_t* flag, cudaStream_t s);
void pack_members(vpg_graph* g, const vpg_records& rec, const int32_t* list, int64_t list_n,
                  int64_t off, void* members, cudaStream_t s, const uint8_t* has_child = nullptr);
void aggregate_range(vpg_graph* g, const void* members, const int64_t* range, int64_t max_count,
                     int S, cudaStream_t s);
// parent links + chunk cost scan (async); chunk table once the host has the total
// linked: k_pack_members + link_children already set every parent
void finalize_operators_async(vpg_graph* g, const vpg_records& rec, cudaStream_t s,
                              const int32_t* parent = nullptr, bool linked = false);
void link_children(vpg_graph* g, const vpg_records& rec, const int32_t* list, int64_t list_n,
                   cudaStream_t s);
// chunk table, descriptors and cluster table on the device (no host sync;
// g->max_cluster must bound the largest cluster)
void finalize_chunks(vpg_graph* g, cudaStream_t s);
// operators.cu: fill g->cluster_id if the build deferred it
void ensure_cluster_ids(const vpg_graph* g, cudaStream_t s);
// shard-local graph from a given cluster partition (records already
// cluster-major, clusters back to back), explicit parents and child flags
void build_local(vpg_graph* g, const vpg_records& rec, int64_t m, const int32_t* cl_size_host,
                 const int32_t* parent, const uint8_t* has_child, int64_t n_halo,
                 const double* halo_ipt, cudaStream_t s);
}  // namespace vpg

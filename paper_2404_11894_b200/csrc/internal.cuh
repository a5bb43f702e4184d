// Cross-translation-unit entry points behind the C ABI (capi.cu).
#pragma once
#include "graph.cuh"

namespace vpg {
void solve(vpg_graph* g, const vpg_records& rec, int32_t iterations, double tol,
           double* residuals, int32_t* performed, cudaStream_t s);
void solve_begin(vpg_graph* g, const vpg_records& rec, int32_t iterations, double tol,
                 cudaStream_t s);
void solve_step(vpg_graph* g, int32_t t, cudaStream_t s);
void solve_control(vpg_graph* g, int32_t t, cudaStream_t s);
void solve_end(vpg_graph* g, double* residuals, int32_t* performed, bool empty, cudaStream_t s);
void splat_arrays(const vpg_paths& P, const double* coeff, const int32_t* clpos, const float4* acc,
                  const float4* dbar, int64_t npix, int spp, int mode, double* image,
                  cudaStream_t s);
void solve_export(const vpg_graph* g, const vpg_records& rec, double* incoming, double* i_bar,
                  cudaStream_t s);
void aggregate_indirect(const vpg_graph* g, const vpg_records& rec, const double* incoming,
                        double* out, cudaStream_t s);
void propagate(const vpg_records& rec, const double* lbar, double* out, int linear, cudaStream_t s);
void export_clusters(const vpg_graph* g, int64_t* cluster_id, int64_t* cl_off, int64_t* members,
                     int64_t* centers, cudaStream_t s);
void export_marginals(const vpg_graph* g, double* p0, double* p1, double* p2, cudaStream_t s);
void export_operators(const vpg_graph* g, int64_t* indptr, int64_t* indices, double* data,
                      double* d_bar, cudaStream_t s);
void splat(const vpg_graph* g, const vpg_records& rec, const vpg_paths& P, int w, int h, int spp,
           int mode, double* image, cudaStream_t s);
void splat_pt(const vpg_paths& P, int w, int h, int spp, double* image, cudaStream_t s);

void trace_image(const vpg_scene& sc, const vpg_trace_cfg& cfg, double* image, cudaStream_t s);
void trace_count(const vpg_scene& sc, const vpg_trace_cfg& cfg, int64_t* counts,
                 const vpg_paths& pth, cudaStream_t s);
void trace_fill(const vpg_scene& sc, const vpg_trace_cfg& cfg, const vpg_records& rec,
                const vpg_paths& pth, cudaStream_t s);
void trace_capture(const vpg_scene& sc, const vpg_trace_cfg& cfg, double* scratch,
                   int64_t capacity, unsigned long long* counter, int64_t* counts,
                   const vpg_paths& pth, cudaStream_t s);
void scatter_records(const double* scratch, int64_t n, const int64_t* rec_start,
                     int64_t path_begin, const vpg_records& out, cudaStream_t s);
int64_t assign_nearest(const double* pos, int64_t n, const double* cpos, int m, const double* lo,
                       const double* hi, int32_t* assign, cudaStream_t s);
struct SplitGroup;
void split_groups_device(vpg_pcg64* state, int32_t* d_ids, const double* d_x, const double* d_y,
                         const double* d_z, const double* d_d0, int64_t n_groups,
                         const int64_t* sizes, const int64_t* centers, const int64_t* cslot_in,
                         int64_t max_size, std::vector<SplitGroup>& groups, int64_t* n_splits,
                         cudaStream_t s);
void choice_device(vpg_pcg64* state, int64_t n, int64_t m, int32_t* d_out, cudaStream_t s);
void codec_rows(bool unpack, uint8_t* packed, int64_t n, int32_t row_bytes,
                const vpg_codec_field* fields, int32_t n_fields, cudaStream_t s);
void reconstruct_paths(const vpg_records& rec, const vpg_paths& pth, const int64_t* ids,
                       int64_t count, double* est, double* diff, cudaStream_t s);
void extra_direct(const vpg_scene& sc, const vpg_records& rec, const vpg_paths& pth, int64_t seed,
                  int n_extra, cudaStream_t s, int64_t path_begin = 0);
}  // namespace vpg

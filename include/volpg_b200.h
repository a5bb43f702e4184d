/*
 * volpg_b200.h — C ABI of libvolpg_b200.so, the sm_100a implementation of the
 * path-graph hot path of arXiv 2404.11894 ("Rendering Participating Media
 * Using Path Graphs").
 *
 * The reference (`volpg` 0.1.0, /root/reference/pkg/src/volpg) is a pure
 * Python/numba package with no FFI of its own; its boundary is the Python API
 * re-exported at pathgraph/__init__.py:1-21 and transport/__init__.py:1-15.
 * Each entry point below is the native half of one of those Python calls; the
 * Python half lives in paper_2404_11894_b200/{pathgraph,transport}/ and is
 * bound with ctypes (paper_2404_11894_b200/_native.py).  The binding a
 * maintainer of the reference would add is shown in INTEGRATION.md.
 *
 * Conventions
 *  - Return value: 0 on success, a negative VPG_E* code on failure; the
 *    message is available from vpg_last_error() (thread-local).
 *  - Pointers documented "device" are CUDA device pointers (the Python layer
 *    passes torch tensor storage); "host" pointers are ordinary memory.
 *  - Every call that launches work takes a `stream` (a cudaStream_t passed as
 *    void*; NULL = legacy default stream) and is stream-ordered.  Calls that
 *    return host data synchronise that stream before returning.
 *  - Layouts follow the reference's RecordSoA / PathSoA exactly
 *    (transport/records.py:27-64): vec3 fields are row-major (n, 3) float64.
 *  - No torch types cross this boundary.
 */
#ifndef VOLPG_B200_H
#define VOLPG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VPG_ABI_VERSION 1

/* error codes (mapped to the reference's exception types by the Python layer) */
#define VPG_OK 0
#define VPG_EINVAL -1    /* ValueError  (clustering.py:34-35, tracer.py:86-87,111-112) */
#define VPG_ECUDA -2     /* RuntimeError: CUDA failure or no device                    */
#define VPG_EDIVERGED -3 /* SolveDivergence (solve.py:28-29,84-90)                     */
#define VPG_ENOMEM -4    /* MemoryError                                                */
#define VPG_ELIMIT -5    /* ValueError: input exceeds a compiled limit                 */

/* ---------------------------------------------------------------- basics */
int vpg_abi_version(void);
const char* vpg_last_error(void);
/* Number of CUDA kernels this library has launched in this process. */
uint64_t vpg_launch_count(void);
/* Bytes this library copied host->device / device->host internally (the
 * build's class statistics, center picks, split-loop staging, exports). */
void vpg_transfer_bytes(uint64_t* h2d, uint64_t* d2h);
/* Per-kernel device timing: when enabled, every launch is bracketed by CUDA
 * events on its stream; vpg_profile_read aggregates (count, total ms) per
 * kernel name ('\n'-separated in `names`).  Diagnostic, used by bench.py. */
void vpg_profile_enable(int32_t on);
int vpg_profile_reset(void);
int vpg_profile_read(char* names, int64_t names_cap, int64_t* counts, double* total_ms,
                     int64_t cap, int64_t* n_kernels);
/* sizeof() of the ABI structs, for binding self-checks:
 * 0 vpg_pcg64, 1 vpg_records, 2 vpg_paths, 3 vpg_graph_info, 4 vpg_scene, 5 vpg_trace_cfg,
 * 6 vpg_graph_views */
size_t vpg_struct_size(int32_t which);
/* Every profiled launch in order: start (ms after the first) and duration. */
int vpg_profile_timeline(char* names, int64_t names_cap, double* start_ms, double* dur_ms,
                         int64_t cap, int64_t* n_launches);

/* ------------------------------------------------- numpy Generator replica
 * Bit-exact replica of numpy.random.Generator(PCG64) for the two calls the
 * reference's clustering makes: Generator.choice(n, m, replace=False)
 * (clustering.py:51 -> numpy tail-shuffle / Floyd branches) and
 * Generator.integers(k) (clustering.py:68).  The state is the one numpy
 * exposes as `bit_generator.state`; the Python layer copies it in and back
 * so a caller's Generator advances exactly as with the reference. */
typedef struct vpg_pcg64 {
  uint64_t state_hi, state_lo; /* 128-bit LCG state */
  uint64_t inc_hi, inc_lo;     /* 128-bit increment (odd) */
  int32_t has_uint32;          /* buffered upper half available */
  uint32_t uinteger;           /* the buffered half */
} vpg_pcg64;

/* out[0..m) = Generator.choice(n, m, replace=False) (host memory). */
/* Generator.choice(n, m, replace=False) (clustering.py:51) with the m picks
 * written to device memory `out` (int32): the tail shuffle's swap targets
 * drawn on the host (exact stream), the swaps resolved on the device. */
int vpg_rng_choice_device(vpg_pcg64* state, int64_t n, int64_t m, int32_t* out, void* stream);
/* The split loop over oversize groups whose members are on the DEVICE (ids
 * and SoA positions / distances, groups back to back, as vpg_split_groups_soa
 * takes them on the host): the first splits' bit rows are computed on the
 * device and the deferred first splits applied there; d_ids ends in final
 * member order.  Outputs as vpg_split_groups_soa (host arrays). */
int vpg_split_groups_device(vpg_pcg64* rng, int32_t* d_ids, const double* d_x, const double* d_y,
                            const double* d_z, const double* d_d0, int64_t n_groups,
                            const int64_t* sizes, const int64_t* centers, const int64_t* cslot,
                            int64_t max_size, int64_t cap_groups, int64_t* out_n_groups,
                            int64_t* out_begin, int64_t* out_size, int64_t* out_center,
                            int64_t* n_splits, void* stream);
int vpg_rng_choice(vpg_pcg64* rng, int64_t n, int64_t m, int64_t* out);
/* out[i] = Generator.integers(k) for i in [0, count) (host memory). */
int vpg_rng_integers(vpg_pcg64* rng, int64_t k, int64_t count, int64_t* out);

/* Host split loop of clustering.py:58-85 (exposed for tests; the device build
 * calls the same code).  Input: groups as CSR over ascending member indices
 * into `pos` (n_pos x 3, float64, host), their centers, the oversize bound
 * `max_size` (= 2K).  Output: the final group list in the reference's order
 * (original groups first, split-off groups appended), as CSR written to
 * caller buffers of capacity `cap_groups` / `n_members`. */
int vpg_split_groups(vpg_pcg64* rng, const double* pos, int64_t n_groups,
                     const int64_t* grp_off, const int64_t* grp_members,
                     const int64_t* grp_center, int64_t max_size,
                     int64_t cap_groups, int64_t* out_n_groups,
                     int64_t* out_off, int64_t* out_members, int64_t* out_center);

/* The split loop on structure-of-arrays input (the sharded build gathers the
 * oversize groups of a class from every shard): ids (n_total, int32, groups
 * back to back, each ascending; reordered in place so every final group is a
 * contiguous ascending run), x/y/z/d0 (member positions and squared distance
 * to the group's center), per group its size, center record id and the slot
 * of the center among its members (-1 if absent).  Out: final groups
 * (originals first, split-off groups appended, clustering.py:58-85) as
 * begin/size/center, capacity cap_groups. */
int vpg_split_groups_soa(vpg_pcg64* rng, int32_t* ids, const double* x, const double* y,
                         const double* z, const double* d0, int64_t n_groups, const int64_t* sizes,
                         const int64_t* centers, const int64_t* cslot, int64_t max_size,
                         int64_t cap_groups, int64_t* out_n_groups, int64_t* out_begin,
                         int64_t* out_size, int64_t* out_center, int64_t* n_splits);

/* Exact nearest center (ties -> lowest index; clustering.py:96-148) of n
 * points against m centers, all device (n x 3, m x 3 float64); bounds (host,
 * 6 doubles: lo xyz, hi xyz) size the hash grid like the class bounding box.
 * assign: n int32 (device).  n_fallback (host, optional): points the
 * neighbourhood search could not decide. */
int vpg_assign_nearest(const double* pos, int64_t n, const double* centers, int64_t m,
                       const double* bounds, int32_t* assign, int64_t* n_fallback, void* stream);

/* ------------------------------------------------------- vertex records
 * Device SoA mirroring RecordSoA (records.py:75-126).  `n` records, stored
 * contiguous per path and depth-ordered (records.py:3-5). */
typedef struct vpg_records {
  int64_t n;
  double* pos;               /* (n,3) */
  double* omega_out;         /* (n,3) toward previous vertex */
  double* normal;            /* (n,3) oriented shading normal (surface) */
  double* coeff;             /* (n,3) sigma_s(x) or albedo */
  double* g;                 /* (n)   HG anisotropy (volume) */
  double* phase_dir;         /* (n,3) */
  double* pdf_phase;         /* (n)   */
  double* pdf_emit_at_phase; /* (n)   */
  double* emit_dir;          /* (n,3) */
  double* pdf_emit;          /* (n)   */
  double* d_emit;            /* (n,3) raw NEE radiance */
  double* d_phase;           /* (n,3) raw phase-hit radiance */
  double* i_pt;              /* (n,3) path-traced incoming indirect */
  double* w_cont;            /* (n,3) Tr/p_t of the arriving segment */
  uint8_t* kind;             /* (n)   0 volume, 1 surface */
  uint8_t* emit_delta;       /* (n)   */
  int32_t* class_id;         /* (n)   medium or surface index */
  int64_t* path_idx;         /* (n)   */
  int32_t* depth;            /* (n)   */
} vpg_records;

/* Device SoA mirroring PathSoA (records.py:144-176). */
typedef struct vpg_paths {
  int64_t n;
  int64_t* pixel_idx;
  int64_t* rec_start;
  int32_t* rec_count;
  double* cam_weight;    /* (n,3) */
  double* d_cam;         /* (n,3) */
  double* direct0;       /* (n,3) */
  double* direct0_nee;   /* (n,3) */
  double* direct0_phase; /* (n,3) */
  double* extra_direct;  /* (n,3) */
  double* pt_estimate;   /* (n,3) */
} vpg_paths;

/* ------------------------------------------------------------ path graph
 * Replaces build_graph (graph.py:56-69) = cluster_points (clustering.py:28-148)
 * + RecordSoA.next_index (records.py:128-140) + compute_marginals
 * (graph.py:94-120) + _build_operators (graph.py:123-168).  The graph keeps
 * its device buffers (cluster-major permutation, dense per-cluster kernel
 * blocks, solve vectors) until vpg_graph_free. */
typedef struct vpg_graph vpg_graph;

typedef struct vpg_graph_info {
  int64_t n_records;
  int64_t n_clusters;
  int64_t nnz;         /* sum over clusters of size^2 (= w_indirect.nnz) */
  int64_t n_classes;
  int64_t n_splits;    /* split-loop iterations performed (clustering.py:58-85) */
  int64_t n_fallback;  /* points resolved by the exact global search (clustering.py:142-147) */
  /* per-stage wall times of the last build when VPG_BUILD_TIMINGS is set: 0 classes,
   * 1 center draw, 2 grid + nearest center, 3 grouping + launch of the part
   * needing no split, 4 host split loop (overlapping the device), 5 split
   * results + wait for the operator kernels, 6 solve chunk table */
  double build_ms[8];
  int64_t n_staged;     /* members of oversize groups sent to the host split loop */
  int64_t split_visits; /* sum of group sizes over all splits (split-loop work) */
} vpg_graph_info;

/* flags for vpg_graph_build */
#define VPG_BUILD_TIMINGS 1       /* record per-stage timings (adds stream syncs) */
#define VPG_BUILD_CLUSTERS_ONLY 2 /* cluster_points only: reads pos, kind, class_id */

/* Cluster the records (class keys kind<<32|class_id, graph.py:59), draw
 * centers with `rng` (advanced in place), and build the aggregation operators.
 * `cluster_size` is K (ValueError if < 1).  The graph borrows `rec`'s device
 * arrays (solve, splat and exports read them): keep them alive and unchanged
 * until vpg_graph_free. */
int vpg_graph_build(const vpg_records* rec, int32_t cluster_size, vpg_pcg64* rng,
                    int32_t flags, void* stream, vpg_graph** out);
/* The same, for records still being uploaded: only pos, kind and class_id
 * must be valid when the call starts; the stream waits on `fields_ready`
 * (a cudaEvent_t) before the build first reads any other field, so the
 * clustering overlaps the rest of the host->device transfer. */
int vpg_graph_build_wait(const vpg_records* rec, int32_t cluster_size, vpg_pcg64* rng,
                         int32_t flags, void* stream, void* fields_ready, vpg_graph** out);
int vpg_graph_info_get(const vpg_graph* g, vpg_graph_info* out);
/* Re-point the graph at the same records (same n) with more fields on the
 * device -- e.g. pdf_phase, which only a 0-iteration solve reads, uploaded
 * after the build. */
int vpg_graph_set_records(vpg_graph* g, const vpg_records* rec);
int vpg_graph_free(vpg_graph* g);

/* Host exports (each synchronises `stream`).  All arrays are in record order.
 * cluster_id: (n) int64; cl_off: (n_clusters+1) int64 offsets into
 * cl_members: (n) int64 member record indices, ascending within a cluster;
 * cl_center: (n_clusters) int64 center record index (clustering.py:23-25). */
int vpg_graph_export_clusters(const vpg_graph* g, int64_t* cluster_id, int64_t* cl_off,
                              int64_t* cl_members, int64_t* cl_center, void* stream);
/* phat_* : (n) float64 marginals (graph.py:94-120). */
int vpg_graph_export_marginals(const vpg_graph* g, double* phat_ind, double* phat_dir_phase,
                               double* phat_dir_emit, void* stream);
/* w_indirect as CSR (graph.py:167): indptr (n+1), indices (nnz), data (nnz);
 * d_bar (n,3) float64 (graph.py:168). Any pointer may be NULL to skip it. */
int vpg_graph_export_operators(const vpg_graph* g, int64_t* indptr, int64_t* indices,
                               double* data, double* d_bar, void* stream);

/* ------------------------------------------------------ shard-local graph
 * Multi-GPU row partition (pathgraph/sharded.py; SURVEY §8e option B): the
 * clusters are partitioned over the shards, every record moves once to the
 * shard owning its cluster, and each shard builds the operators of its own
 * clusters with this call.  `rec` (device, n rows) is already cluster-major:
 * the n_clusters clusters lie back to back with cl_size[k] (host) members in
 * ascending global record order, so marginals, kernel blocks and D-bar are
 * computed exactly as by vpg_graph_build (graph.py:94-168).  Continuation
 * edges are explicit because a record's parent (record r-1 of the same path,
 * records.py:128-140) may live on another shard:
 *   parent[q]    (n, device) local row of q's parent, -1 for a path's first
 *                record, or n + h: halo slot h (the parent is remote)
 *   has_child[q] (n, device u8) 1 if q has a continuation child anywhere
 *   halo_ipt     (n_halo x 3 fp64, device) i_pt of each halo slot's parent
 *                (its I_0, solve.py:72)
 * The solve then runs as vpg_solve_begin, per iteration vpg_solve_step ->
 * (the caller sends halo slots n.. of the output I vector to their owners,
 * writes the received values into its own rows, and max-reduces the 7
 * residual words red[t*8 .. t*8+6] and, once, term_max[0..2] over all
 * shards) -> vpg_solve_control, and finally vpg_solve_end.  On one shard
 * (n_halo = 0, nothing to exchange) this is exactly vpg_solve. */
int vpg_graph_build_local(const vpg_records* rec, int64_t n_clusters, const int32_t* cl_size,
                          const int32_t* parent, const uint8_t* has_child, int64_t n_halo,
                          const double* halo_ipt, void* stream, vpg_graph** out);

/* Device pointers into a graph (read-only unless stated; valid until
 * vpg_graph_free).  float* vectors are float4 per row (xyz = RGB).
 * ibuf[t&1] is iteration t's input I, ibuf[(t+1)&1] its output (halo slots
 * n .. n+n_halo-1 included); acc = W*I; red[t*8 + 0..5] = float bits of the
 * residual maxima, red[t*8 + 6] = NaN channel bits (writable between step
 * and control); term_max[0..2] writable after the build. */
typedef struct vpg_graph_views {
  int64_t n, m, n_halo;
  int32_t *perm, *clpos, *cluster_id, *cl_off, *cl_size, *cl_center, *ref_of, *internal_of;
  float *i0, *ibuf[2], *acc[2], *dbar;
  float* term_max;
  uint32_t* red;
  int32_t* ctl;
  int32_t performed;
  int32_t _pad;
} vpg_graph_views;
int vpg_graph_views_get(const vpg_graph* g, vpg_graph_views* views);

/* ----------------------------------------------------------------- solve
 * Replaces solve (solve.py:64-98): device-resident fixed point
 * I <- P A+ I + P Ao D with the residual, tol break and 3-growth divergence
 * rule evaluated on the device.  residuals: host, capacity `iterations`.
 * Returns VPG_EDIVERGED (after filling residuals/performed) on divergence. */
int vpg_solve(vpg_graph* g, int32_t iterations, double tol, double* residuals,
              int32_t* performed, void* stream);
/* The pieces of vpg_solve, for shard-local graphs (see vpg_graph_build_local). */
int vpg_solve_begin(vpg_graph* g, int32_t iterations, double tol, void* stream);
int vpg_solve_step(vpg_graph* g, int32_t t, void* stream);
int vpg_solve_control(vpg_graph* g, int32_t t, void* stream);
int vpg_solve_end(vpg_graph* g, double* residuals, int32_t* performed, void* stream);
/* incoming, i_bar: (n,3) float64 host, record order (SolveResult fields). */
int vpg_solve_export(const vpg_graph* g, double* incoming, double* i_bar, void* stream);

/* aggregate_indirect (operators.py:17-19): out = coeff * (W @ incoming).
 * propagate / propagate_linear (operators.py:27-47): out[r] = w_cont[r+1] *
 * l_bar[r+1] on continuation edges, i_pt (linear=0) or 0 (linear=1) elsewhere.
 * All (n,3) float64 device arrays in record order. */
int vpg_aggregate_indirect(const vpg_graph* g, const double* incoming, double* out, void* stream);
int vpg_propagate(const vpg_records* rec, const double* l_bar, double* out, int32_t linear,
                  void* stream);

/* ----------------------------------------------------------------- splat
 * Replaces splat_output (solve.py:101-132). direct_mode: 0 = direct0,
 * 1 = extra_direct, 2 = aggregated D-bar.  image: (height,width,3) float64
 * device.  Uses the last solve's i_bar. */
#define VPG_DIRECT_PT 0
#define VPG_DIRECT_EXTRA 1
#define VPG_DIRECT_AGGREGATED 2
int vpg_splat(const vpg_graph* g, const vpg_paths* paths, int32_t width, int32_t height,
              int32_t spp, int32_t direct_mode, double* image, void* stream);
/* splat_output over explicit arrays (a shard's pixel range): path p's first
 * record r0 = paths->rec_start[p] reads coeff[r0] (fp64 x3) and the float4
 * acc / dbar at index clpos[r0].  n_pixels * spp == paths->n. */
int vpg_splat_arrays(const vpg_paths* paths, const double* coeff, const int32_t* clpos,
                     const float* acc4, const float* dbar4, int64_t n_pixels, int32_t spp,
                     int32_t direct_mode, double* image, void* stream);
/* splat_pt_image (records.py:259-265): per-pixel mean of pt_estimate. */
int vpg_splat_pt(const vpg_paths* paths, int32_t width, int32_t height, int32_t spp,
                 double* image, void* stream);

/* ---------------------------------------------------------------- tracer
 * Packed scene (flatten.py:87-195 equivalent), passed by value to kernels. */
#define VPG_MAX_SURF 32
#define VPG_MAX_EMIT 16
#define VPG_MAX_MED 8
typedef struct vpg_scene {
  int32_t n_surf, n_emit, n_med, width, height, _pad0;
  int32_t surf_type[VPG_MAX_SURF];  /* 0 sphere, 1 box, 2 quad */
  int32_t mat_type[VPG_MAX_SURF];   /* 0 lambertian, 1 black, 2 emitter */
  int32_t emitter_id[VPG_MAX_SURF];
  double surf_params[VPG_MAX_SURF][9];
  double albedo[VPG_MAX_SURF][3];
  int32_t em_type[VPG_MAX_EMIT];    /* 0 point, 1 area, 2 directional */
  double em_value[VPG_MAX_EMIT][3];
  double em_pos[VPG_MAX_EMIT][3];   /* point position / unit travel direction */
  double em_quad[VPG_MAX_EMIT][9];
  double em_normal[VPG_MAX_EMIT][3];
  double em_area[VPG_MAX_EMIT];
  int32_t med_kind[VPG_MAX_MED];    /* 0 homogeneous, 1 grid */
  int32_t grid_dims[VPG_MAX_MED][3];/* nx, ny, nz */
  double med_sigma_t[VPG_MAX_MED][3];
  double med_sigma_s[VPG_MAX_MED][3];
  double med_g[VPG_MAX_MED];
  double med_bounds[VPG_MAX_MED][6];
  double med_majorant[VPG_MAX_MED];
  double med_scale[VPG_MAX_MED];
  int64_t grid_offset[VPG_MAX_MED];
  const float* grid_data;           /* device, concatenated (z,y,x) float32 volumes */
  double cam[15];                   /* origin, forward, right, up, tan_half, W, H */
} vpg_scene;

typedef struct vpg_trace_cfg {
  int32_t spp;
  int32_t max_depth;
  int32_t rr_start;
  int32_t _pad;
  double rr_floor;
  int64_t seed;
  int64_t path_begin; /* first path id of this launch (multi-GPU row partition) */
  int64_t path_count; /* number of paths (global ids path_begin..) */
} vpg_trace_cfg;

/* Record-free render (render_image_kernel, kernels.py:433-460): image
 * (height,width,3) float64 device. */
int vpg_trace_image(const vpg_scene* scene, const vpg_trace_cfg* cfg, double* image, void* stream);
/* Pass 1 (count_records_kernel, kernels.py:463-479): counts (path_count) int64
 * device, plus the path-table estimates. */
int vpg_trace_count(const vpg_scene* scene, const vpg_trace_cfg* cfg, int64_t* counts,
                    const vpg_paths* paths, void* stream);
/* Pass 2 (fill_records_kernel, kernels.py:482-496): writes records at
 * paths->rec_start offsets (relative to `rec`), and the path table. */
int vpg_trace_fill(const vpg_scene* scene, const vpg_trace_cfg* cfg, const vpg_records* rec,
                   const vpg_paths* paths, void* stream);
/* Single-pass capture (replaces pass 1 + pass 2): every path is traced once
 * and its records go to scratch slots (capacity `capacity`) claimed through
 * the device `counter`; counts (path_count) and the path table are written as
 * in pass 1.  If *counter > capacity afterwards, records were dropped: retry
 * with capacity >= *counter (deterministic).  The scratch (device) holds one
 * record per slot, VPG_SCRATCH_DOUBLES doubles each (a slot-major layout, so
 * a path's stores land in its own slot).  vpg_scatter_records then writes the
 * n = *counter scratch records, in path order (row = rec_start[path -
 * path_begin] + depth), into the SoA `out`, and runs the backward i_pt sweep
 * (kernels.py:393-408) over them there.  Any max_depth. */
#define VPG_SCRATCH_DOUBLES 40
int vpg_trace_capture(const vpg_scene* scene, const vpg_trace_cfg* cfg, double* scratch,
                      int64_t capacity, uint64_t* counter, int64_t* counts, const vpg_paths* paths,
                      void* stream);
int vpg_scatter_records(const double* scratch, int64_t n, const int64_t* rec_start,
                        int64_t path_begin, const vpg_records* out, void* stream);
/* ------------------------------------------------------------ VPGR codec
 * Packed rows (a VPGR dump's record or path block, records.py:191-256) <->
 * per-field device arrays, on the device: `packed` (device) holds n rows of
 * row_bytes; field f occupies bytes [offset, offset+bytes) of a row and
 * fields[f].ptr (device) is its array (row i at ptr + i*bytes).  Loading a
 * dump is one host->device copy of the block plus vpg_unpack_rows; saving
 * from the device is vpg_pack_rows plus one device->host copy. */
#define VPG_CODEC_MAX_FIELDS 24
typedef struct vpg_codec_field {
  int32_t offset;
  int32_t bytes;
  void* ptr;
} vpg_codec_field;
int vpg_unpack_rows(const void* packed, int64_t n, int32_t row_bytes,
                    const vpg_codec_field* fields, int32_t n_fields, void* stream);
int vpg_pack_rows(void* packed, int64_t n, int32_t row_bytes, const vpg_codec_field* fields,
                  int32_t n_fields, void* stream);

/* extra_direct_kernel (kernels.py:499-553). */
int vpg_extra_direct(const vpg_scene* scene, const vpg_records* rec, const vpg_paths* paths,
                     int64_t seed, int32_t n_extra, void* stream);

/* Frees the library's cached device memory (scratch buffers and the free
 * part of the stream-ordered pool) after a device synchronisation; graphs
 * alive keep their own buffers. */
int vpg_release_cached(void);

/* vpg_extra_direct over a slice of the frame's path table whose first row is
 * path `path_begin` of the frame (a shard's pixel range): the per-path
 * streams are keyed by the frame's path index (kernels.py:532-536). */
int vpg_extra_direct_range(const vpg_scene* scene, const vpg_records* rec, const vpg_paths* paths,
                           int64_t path_begin, int64_t seed, int32_t n_extra, void* stream);

/* reconstruct_path_estimate (transport/reconstruct.py:52-72) for `count`
 * paths: path_ids (device int64, or NULL for paths 0..count-1); outputs
 * estimate (count,3) float64 = d_cam + the backward walk over the path's
 * records, and max_ipt_diff (count,) float64 = max |stored i_pt - recomputed
 * incoming| (device). */
int vpg_reconstruct_paths(const vpg_records* rec, const vpg_paths* paths, const int64_t* path_ids,
                          int64_t count, double* estimate, double* max_ipt_diff, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* VOLPG_B200_H */

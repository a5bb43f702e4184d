// extern "C" entry points of libvolpg_b200.so (declared in include/volpg_b200.h).
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "host_rng.hpp"
#include "internal.cuh"

namespace vpg {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
std::once_flag g_pool_once;
int g_sm_count = 0;
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int sm_count() {
  if (g_sm_count == 0) {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      g_sm_count = v;
    else
      g_sm_count = 148;
  }
  return g_sm_count;
}

void* dalloc(size_t bytes, cudaStream_t s) {
  std::call_once(g_pool_once, [] {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  });
  void* p = nullptr;
  const cudaError_t e = cudaMallocAsync(&p, bytes ? bytes : 16, s);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(e == cudaErrorMemoryAllocation ? VPG_ENOMEM : VPG_ECUDA,
                std::string("device allocation of ") + std::to_string(bytes) +
                    " bytes failed: " + cudaGetErrorString(e));
  }
  return p;
}

void dfree(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}

}  // namespace vpg

using vpg::guarded;

static cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

extern "C" {

int vpg_abi_version(void) { return VPG_ABI_VERSION; }
const char* vpg_last_error(void) { return vpg::g_last_error.c_str(); }
uint64_t vpg_launch_count(void) { return vpg::g_launches.load(); }

size_t vpg_struct_size(int32_t which) {
  switch (which) {
    case 0: return sizeof(vpg_pcg64);
    case 1: return sizeof(vpg_records);
    case 2: return sizeof(vpg_paths);
    case 3: return sizeof(vpg_graph_info);
    case 4: return sizeof(vpg_scene);
    case 5: return sizeof(vpg_trace_cfg);
    default: return 0;
  }
}

int vpg_rng_choice(vpg_pcg64* rng, int64_t n, int64_t m, int64_t* out) {
  return guarded([&] {
    VPG_REQUIRE(n >= 0 && m >= 0 && m <= n, VPG_EINVAL,
                "Cannot take a larger sample than population when replace is False");
    vpg::Pcg64 g(*rng);
    vpg::rng_choice(g, n, m, out);
    g.store(rng);
  });
}

int vpg_rng_integers(vpg_pcg64* rng, int64_t k, int64_t count, int64_t* out) {
  return guarded([&] {
    VPG_REQUIRE(k >= 1, VPG_EINVAL, "high <= 0");
    vpg::Pcg64 g(*rng);
    for (int64_t i = 0; i < count; ++i) out[i] = int64_t(g.bounded(uint64_t(k - 1)));
    g.store(rng);
  });
}

int vpg_split_groups(vpg_pcg64* rng, const double* pos, int64_t n_groups, const int64_t* grp_off,
                     const int64_t* grp_members, const int64_t* grp_center, int64_t max_size,
                     int64_t cap_groups, int64_t* out_n_groups, int64_t* out_off,
                     int64_t* out_members, int64_t* out_center) {
  return guarded([&] {
    vpg::Pcg64 g(*rng);
    std::vector<int64_t> over;
    std::vector<std::vector<int64_t>> groups;
    std::vector<int64_t> centers;
    for (int64_t c = 0; c < n_groups; ++c) {
      if (grp_off[c + 1] - grp_off[c] > max_size) {
        over.push_back(c);
        groups.emplace_back(grp_members + grp_off[c], grp_members + grp_off[c + 1]);
        centers.push_back(grp_center[c]);
      }
    }
    vpg::split_oversize(g, groups, centers, max_size,
                        [&](int64_t id) { return pos + size_t(id) * 3; });
    const int64_t total = n_groups + int64_t(groups.size()) - int64_t(over.size());
    VPG_REQUIRE(total <= cap_groups, VPG_ELIMIT, "output group capacity exceeded");
    int64_t w = 0, o = 0;
    size_t next = 0;
    auto emit = [&](const int64_t* b, const int64_t* e, int64_t center) {
      out_off[w] = o;
      for (const int64_t* p = b; p != e; ++p) out_members[o++] = *p;
      out_center[w++] = center;
    };
    for (int64_t c = 0; c < n_groups; ++c) {
      if (next < over.size() && over[next] == c) {
        emit(groups[next].data(), groups[next].data() + groups[next].size(), centers[next]);
        ++next;
      } else {
        emit(grp_members + grp_off[c], grp_members + grp_off[c + 1], grp_center[c]);
      }
    }
    for (size_t k = over.size(); k < groups.size(); ++k)
      emit(groups[k].data(), groups[k].data() + groups[k].size(), centers[k]);
    out_off[w] = o;
    *out_n_groups = w;
    g.store(rng);
  });
}

int vpg_graph_build(const vpg_records* rec, int32_t cluster_size, vpg_pcg64* rng, int32_t flags,
                    void* stream, vpg_graph** out) {
  *out = nullptr;
  vpg_graph* g = new vpg_graph();
  const int rc = guarded([&] {
    g->stream = as_stream(stream);
    g->rec = *rec;
    vpg::build_clusters(g, *rec, cluster_size, rng, (flags & VPG_BUILD_TIMINGS) != 0, g->stream);
    if (!(flags & VPG_BUILD_CLUSTERS_ONLY)) vpg::build_operators(g, *rec, g->stream);
    if (flags & VPG_BUILD_TIMINGS) VPG_CUDA(cudaStreamSynchronize(g->stream));
    g->info.n_records = g->n;
    g->info.n_clusters = g->m;
    g->info.nnz = g->nnz;
  });
  if (rc != VPG_OK) {
    delete g;
    return rc;
  }
  *out = g;
  return VPG_OK;
}

int vpg_graph_info_get(const vpg_graph* g, vpg_graph_info* out) {
  return guarded([&] { *out = g->info; });
}

int vpg_graph_free(vpg_graph* g) {
  return guarded([&] { delete g; });
}

int vpg_graph_export_clusters(const vpg_graph* g, int64_t* cluster_id, int64_t* cl_off,
                              int64_t* cl_members, int64_t* cl_center, void* stream) {
  return guarded([&] {
    vpg::export_clusters(g, cluster_id, cl_off, cl_members, cl_center, as_stream(stream));
  });
}

int vpg_graph_export_marginals(const vpg_graph* g, double* a, double* b, double* c, void* stream) {
  return guarded([&] { vpg::export_marginals(g, a, b, c, as_stream(stream)); });
}

int vpg_graph_export_operators(const vpg_graph* g, int64_t* indptr, int64_t* indices, double* data,
                               double* d_bar, void* stream) {
  return guarded([&] { vpg::export_operators(g, indptr, indices, data, d_bar, as_stream(stream)); });
}

int vpg_solve(vpg_graph* g, int32_t iterations, double tol, double* residuals, int32_t* performed,
              void* stream) {
  return guarded([&] {
    vpg::solve(g, g->rec, iterations, tol, residuals, performed, as_stream(stream));
  });
}

int vpg_solve_export(const vpg_graph* g, double* incoming, double* i_bar, void* stream) {
  return guarded([&] { vpg::solve_export(g, g->rec, incoming, i_bar, as_stream(stream)); });
}

int vpg_aggregate_indirect(const vpg_graph* g, const double* incoming, double* out, void* stream) {
  return guarded([&] { vpg::aggregate_indirect(g, g->rec, incoming, out, as_stream(stream)); });
}

int vpg_propagate(const vpg_records* rec, const double* l_bar, double* out, int32_t linear,
                  void* stream) {
  return guarded([&] { vpg::propagate(*rec, l_bar, out, linear, as_stream(stream)); });
}

int vpg_splat(const vpg_graph* g, const vpg_paths* paths, int32_t width, int32_t height,
              int32_t spp, int32_t direct_mode, double* image, void* stream) {
  return guarded([&] {
    vpg::splat(g, g->rec, *paths, width, height, spp, direct_mode, image, as_stream(stream));
  });
}

int vpg_splat_pt(const vpg_paths* paths, int32_t width, int32_t height, int32_t spp, double* image,
                 void* stream) {
  return guarded([&] { vpg::splat_pt(*paths, width, height, spp, image, as_stream(stream)); });
}

int vpg_trace_image(const vpg_scene* scene, const vpg_trace_cfg* cfg, double* image, void* stream) {
  return guarded([&] { vpg::trace_image(*scene, *cfg, image, as_stream(stream)); });
}

int vpg_trace_count(const vpg_scene* scene, const vpg_trace_cfg* cfg, int64_t* counts,
                    const vpg_paths* paths, void* stream) {
  return guarded([&] { vpg::trace_count(*scene, *cfg, counts, *paths, as_stream(stream)); });
}

int vpg_trace_fill(const vpg_scene* scene, const vpg_trace_cfg* cfg, const vpg_records* rec,
                   const vpg_paths* paths, void* stream) {
  return guarded([&] { vpg::trace_fill(*scene, *cfg, *rec, *paths, as_stream(stream)); });
}

int vpg_extra_direct(const vpg_scene* scene, const vpg_records* rec, const vpg_paths* paths,
                     int64_t seed, int32_t n_extra, void* stream) {
  return guarded([&] { vpg::extra_direct(*scene, *rec, *paths, seed, n_extra, as_stream(stream)); });
}

}  // extern "C"

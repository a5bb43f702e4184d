// extern "C" entry points of libvolpg_b200.so (declared in include/volpg_b200.h).
#include <atomic>
#include <map>
#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "host_rng.hpp"
#include "internal.cuh"

namespace vpg {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }

namespace {
struct ProfEntry {
  std::string name;
  cudaEvent_t start, stop;
};
std::atomic<bool> g_profiling{false};
std::mutex g_prof_mu;
std::vector<ProfEntry> g_prof;
}  // namespace

bool profiling() { return g_profiling.load(std::memory_order_relaxed); }

int prof_begin(const char* name, cudaStream_t s) {
  ProfEntry e{name, nullptr, nullptr};
  if (cudaEventCreate(&e.start) != cudaSuccess || cudaEventCreate(&e.stop) != cudaSuccess) return -1;
  cudaEventRecord(e.start, s);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.push_back(e);
  return int(g_prof.size()) - 1;
}

void prof_end(int token, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (token >= 0 && token < int(g_prof.size())) cudaEventRecord(g_prof[token].stop, s);
}
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

namespace {
std::atomic<uint64_t> g_h2d{0}, g_d2h{0};
}
void count_transfer(uint64_t h2d, uint64_t d2h) {
  g_h2d.fetch_add(h2d, std::memory_order_relaxed);
  g_d2h.fetch_add(d2h, std::memory_order_relaxed);
}

namespace {
constexpr int kMaxDevices = 64;
int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  return dev;
}
std::atomic<int> g_sm_counts[kMaxDevices];
std::once_flag g_pool_once[kMaxDevices];
std::mutex g_attr_mu;
std::map<std::pair<int, const void*>, size_t> g_smem_attr;
}  // namespace

// per device: a process may drive several GPUs (one context per device)
int sm_count() {
  const int dev = current_device();
  int v = g_sm_counts[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    g_sm_counts[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

void ensure_dynamic_smem(const void* func, size_t bytes) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_attr_mu);
  size_t& have = g_smem_attr[{dev, func}];
  if (bytes > have) {
    VPG_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    have = bytes;
  }
}

void* dalloc(size_t bytes, cudaStream_t s) {
  const int dev = current_device();
  std::call_once(g_pool_once[dev], [dev] {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
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

namespace {
std::mutex g_scratch_mu;
std::map<std::pair<cudaStream_t, std::string>, std::pair<void*, size_t>>& g_scratch() {
  static std::map<std::pair<cudaStream_t, std::string>, std::pair<void*, size_t>> m;
  return m;
}
}  // namespace

// Frees every scratch buffer and returns the stream-ordered pool's free
// memory to the device (after a device sync): for callers that need the HBM
// for something else between builds.
void release_cached() {
  VPG_CUDA(cudaDeviceSynchronize());
  {
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    for (auto& kv : g_scratch())
      if (kv.second.first) cudaFree(kv.second.first);
    g_scratch().clear();
  }
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
    VPG_CUDA(cudaMemPoolTrimTo(pool, 0));
}

void* scratch(cudaStream_t s, const char* tag, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_scratch_mu);
  auto& e = g_scratch()[{s, std::string(tag)}];
  if (e.second < bytes) {
    if (e.first) {
      VPG_CUDA(cudaStreamSynchronize(s));  // the old buffer may still be in use
      VPG_CUDA(cudaFree(e.first));
      e.first = nullptr;
    }
    const size_t cap = bytes + bytes / 8;
    void* p = nullptr;
    const cudaError_t err = cudaMalloc(&p, cap);
    if (err != cudaSuccess) {
      cudaGetLastError();
      e.second = 0;
      throw Error(VPG_ENOMEM, std::string("scratch allocation failed: ") + cudaGetErrorString(err));
    }
    e.first = p;
    e.second = cap;
  }
  return e.first;
}

namespace {
std::map<void*, size_t>& g_host_cap() {
  static std::map<void*, size_t> caps;
  return caps;
}
std::mutex g_host_mu;
std::vector<std::pair<size_t, void*>> g_host_free;  // (capacity, pointer)
}  // namespace

void* halloc(size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_host_mu);
    size_t best = g_host_free.size();
    for (size_t i = 0; i < g_host_free.size(); ++i)
      if (g_host_free[i].first >= bytes &&
          (best == g_host_free.size() || g_host_free[i].first < g_host_free[best].first))
        best = i;
    if (best < g_host_free.size() && g_host_free[best].first <= 4 * bytes + (1 << 20)) {
      void* p = g_host_free[best].second;
      g_host_free.erase(g_host_free.begin() + best);
      return p;
    }
  }
  const size_t cap = bytes < (1 << 20) ? (1 << 20) : bytes + bytes / 4;
  void* p = nullptr;
  if (cudaMallocHost(&p, cap) != cudaSuccess) {
    cudaGetLastError();
    throw Error(VPG_ENOMEM, "pinned host allocation failed");
  }
  std::lock_guard<std::mutex> lk(g_host_mu);
  g_host_cap()[p] = cap;
  return p;
}

void hfree(void* p, size_t) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_host_mu);
  g_host_free.emplace_back(g_host_cap()[p], p);
}

}  // namespace vpg

using vpg::guarded;

static cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

extern "C" {

int vpg_abi_version(void) { return VPG_ABI_VERSION; }
const char* vpg_last_error(void) { return vpg::g_last_error.c_str(); }
uint64_t vpg_launch_count(void) { return vpg::g_launches.load(); }
void vpg_transfer_bytes(uint64_t* h2d, uint64_t* d2h) {
  *h2d = vpg::g_h2d.load();
  *d2h = vpg::g_d2h.load();
}

size_t vpg_struct_size(int32_t which) {
  switch (which) {
    case 0: return sizeof(vpg_pcg64);
    case 1: return sizeof(vpg_records);
    case 2: return sizeof(vpg_paths);
    case 3: return sizeof(vpg_graph_info);
    case 4: return sizeof(vpg_scene);
    case 5: return sizeof(vpg_trace_cfg);
    case 6: return sizeof(vpg_graph_views);
    default: return 0;
  }
}

void vpg_profile_enable(int32_t on) { vpg::g_profiling.store(on != 0); }

int vpg_profile_reset(void) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(vpg::g_prof_mu);
    for (auto& e : vpg::g_prof) {
      cudaEventDestroy(e.start);
      cudaEventDestroy(e.stop);
    }
    vpg::g_prof.clear();
  });
}

int vpg_profile_timeline(char* names, int64_t names_cap, double* start_ms, double* dur_ms,
                         int64_t cap, int64_t* n_launches) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(vpg::g_prof_mu);
    std::string joined;
    int64_t k = 0;
    for (auto& e : vpg::g_prof) {
      VPG_CUDA(cudaEventSynchronize(e.stop));
      float t0 = 0.f, d = 0.f;
      VPG_CUDA(cudaEventElapsedTime(&t0, vpg::g_prof.front().start, e.start));
      VPG_CUDA(cudaEventElapsedTime(&d, e.start, e.stop));
      if (k < cap) {
        start_ms[k] = t0;
        dur_ms[k] = d;
        joined += e.name;
        joined += '\n';
      }
      ++k;
    }
    *n_launches = k;
    VPG_REQUIRE(int64_t(joined.size()) < names_cap, VPG_ELIMIT, "profile name buffer too small");
    memcpy(names, joined.c_str(), joined.size() + 1);
  });
}

int vpg_profile_read(char* names, int64_t names_cap, int64_t* counts, double* total_ms,
                     int64_t cap, int64_t* n_kernels) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(vpg::g_prof_mu);
    std::vector<std::string> keys;
    std::vector<int64_t> cnt;
    std::vector<double> ms;
    for (auto& e : vpg::g_prof) {
      VPG_CUDA(cudaEventSynchronize(e.stop));
      float t = 0.f;
      VPG_CUDA(cudaEventElapsedTime(&t, e.start, e.stop));
      size_t k = 0;
      while (k < keys.size() && keys[k] != e.name) ++k;
      if (k == keys.size()) {
        keys.push_back(e.name);
        cnt.push_back(0);
        ms.push_back(0.0);
      }
      cnt[k] += 1;
      ms[k] += t;
    }
    *n_kernels = int64_t(keys.size());
    std::string joined;
    for (size_t k = 0; k < keys.size() && int64_t(k) < cap; ++k) {
      counts[k] = cnt[k];
      total_ms[k] = ms[k];
      joined += keys[k];
      joined += '\n';
    }
    VPG_REQUIRE(int64_t(joined.size()) < names_cap, VPG_ELIMIT, "profile name buffer too small");
    memcpy(names, joined.c_str(), joined.size() + 1);
  });
}

int vpg_rng_choice_device(vpg_pcg64* state, int64_t n, int64_t m, int32_t* out, void* stream) {
  return guarded([&] { vpg::choice_device(state, n, m, out, as_stream(stream)); });
}

int vpg_split_groups_device(vpg_pcg64* rng, int32_t* d_ids, const double* d_x, const double* d_y,
                            const double* d_z, const double* d_d0, int64_t n_groups,
                            const int64_t* sizes, const int64_t* centers, const int64_t* cslot,
                            int64_t max_size, int64_t cap_groups, int64_t* out_n_groups,
                            int64_t* out_begin, int64_t* out_size, int64_t* out_center,
                            int64_t* n_splits, void* stream) {
  return guarded([&] {
    std::vector<vpg::SplitGroup> groups;
    vpg::split_groups_device(rng, d_ids, d_x, d_y, d_z, d_d0, n_groups, sizes, centers, cslot,
                             max_size, groups, n_splits, as_stream(stream));
    VPG_REQUIRE(int64_t(groups.size()) <= cap_groups, VPG_ELIMIT, "output group capacity exceeded");
    for (size_t k = 0; k < groups.size(); ++k) {
      out_begin[k] = groups[k].begin;
      out_size[k] = groups[k].size;
      out_center[k] = groups[k].center;
    }
    *out_n_groups = int64_t(groups.size());
  });
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
    std::vector<int32_t> ids;
    std::vector<double> xyz, cxyz;
    std::vector<vpg::SplitGroup> groups;
    for (int64_t c = 0; c < n_groups; ++c) {
      const int64_t size = grp_off[c + 1] - grp_off[c];
      if (size <= max_size) continue;
      over.push_back(c);
      groups.push_back(vpg::SplitGroup{int64_t(ids.size()), size, grp_center[c]});
      for (int a = 0; a < 3; ++a) cxyz.push_back(pos[grp_center[c] * 3 + a]);
      for (int64_t t = grp_off[c]; t < grp_off[c + 1]; ++t) {
        ids.push_back(int32_t(grp_members[t]));
        for (int a = 0; a < 3; ++a) xyz.push_back(pos[grp_members[t] * 3 + a]);
      }
    }
    vpg::split_oversize(g, ids.data(), xyz.data(), ids.size(), groups, max_size, cxyz.data());
    const int64_t total = n_groups + int64_t(groups.size()) - int64_t(over.size());
    VPG_REQUIRE(total <= cap_groups, VPG_ELIMIT, "output group capacity exceeded");
    int64_t w = 0, o = 0;
    size_t next = 0;
    auto emit = [&](const int64_t* b, const int64_t* e, int64_t center) {
      out_off[w] = o;
      for (const int64_t* p = b; p != e; ++p) out_members[o++] = *p;
      out_center[w++] = center;
    };
    auto emit_split = [&](const vpg::SplitGroup& sg) {
      std::vector<int64_t> wide(ids.begin() + sg.begin, ids.begin() + sg.begin + sg.size);
      emit(wide.data(), wide.data() + wide.size(), sg.center);
    };
    for (int64_t c = 0; c < n_groups; ++c) {
      if (next < over.size() && over[next] == c)
        emit_split(groups[next++]);
      else
        emit(grp_members + grp_off[c], grp_members + grp_off[c + 1], grp_center[c]);
    }
    for (size_t k = over.size(); k < groups.size(); ++k) emit_split(groups[k]);
    out_off[w] = o;
    *out_n_groups = w;
    g.store(rng);
  });
}

int vpg_graph_build_wait(const vpg_records* rec, int32_t cluster_size, vpg_pcg64* rng,
                         int32_t flags, void* stream, void* fields_ready, vpg_graph** out) {
  *out = nullptr;
  vpg_graph* g = new vpg_graph();
  const int rc = guarded([&] {
    g->stream = as_stream(stream);
    g->rec = *rec;
    vpg::build_graph(g, *rec, cluster_size, rng, (flags & VPG_BUILD_TIMINGS) != 0,
                     !(flags & VPG_BUILD_CLUSTERS_ONLY), g->stream,
                     static_cast<cudaEvent_t>(fields_ready));
    g->info.n_records = g->n;
    g->info.n_clusters = g->m;
    if (!g->tot_pending) g->info.nnz = g->nnz;
  });
  if (rc != VPG_OK) {
    delete g;
    return rc;
  }
  *out = g;
  return VPG_OK;
}

int vpg_unpack_rows(const void* packed, int64_t n, int32_t row_bytes,
                    const vpg_codec_field* fields, int32_t n_fields, void* stream) {
  return guarded([&] {
    vpg::codec_rows(true, static_cast<uint8_t*>(const_cast<void*>(packed)), n, row_bytes, fields,
                    n_fields, as_stream(stream));
  });
}

int vpg_pack_rows(void* packed, int64_t n, int32_t row_bytes, const vpg_codec_field* fields,
                  int32_t n_fields, void* stream) {
  return guarded([&] {
    vpg::codec_rows(false, static_cast<uint8_t*>(packed), n, row_bytes, fields, n_fields,
                    as_stream(stream));
  });
}

int vpg_split_groups_soa(vpg_pcg64* rng, int32_t* ids, const double* x, const double* y,
                         const double* z, const double* d0, int64_t n_groups, const int64_t* sizes,
                         const int64_t* centers, const int64_t* cslot, int64_t max_size,
                         int64_t cap_groups, int64_t* out_n_groups, int64_t* out_begin,
                         int64_t* out_size, int64_t* out_center, int64_t* n_splits) {
  return guarded([&] {
    vpg::Pcg64 g(*rng);
    std::vector<vpg::SplitGroup> groups(static_cast<size_t>(n_groups));
    std::vector<int64_t> slot(static_cast<size_t>(n_groups));
    int64_t total = 0;
    for (int64_t k = 0; k < n_groups; ++k) {
      groups[k] = vpg::SplitGroup{total, sizes[k], centers[k]};
      slot[k] = cslot[k];
      total += sizes[k];
    }
    std::vector<double> X(x, x + total), Y(y, y + total), Z(z, z + total), D(d0, d0 + total);
    const int64_t n = vpg::split_oversize_soa(
        g, vpg::SplitMembers{ids, X.data(), Y.data(), Z.data(), D.data()}, groups, slot, max_size);
    VPG_REQUIRE(int64_t(groups.size()) <= cap_groups, VPG_ELIMIT, "output group capacity exceeded");
    for (size_t k = 0; k < groups.size(); ++k) {
      out_begin[k] = groups[k].begin;
      out_size[k] = groups[k].size;
      out_center[k] = groups[k].center;
    }
    *out_n_groups = int64_t(groups.size());
    *n_splits = n;
    g.store(rng);
  });
}

int vpg_assign_nearest(const double* pos, int64_t n, const double* centers, int64_t m,
                       const double* bounds, int32_t* assign, int64_t* n_fallback, void* stream) {
  return guarded([&] {
    VPG_REQUIRE(m >= 1 && m < (int64_t(1) << 31) && n < (int64_t(1) << 31), VPG_ELIMIT,
                "assign_nearest: sizes out of range");
    const int64_t fb = vpg::assign_nearest(pos, n, centers, int(m), bounds, bounds + 3, assign,
                                           as_stream(stream));
    if (n_fallback) *n_fallback = fb;
  });
}

int vpg_graph_build(const vpg_records* rec, int32_t cluster_size, vpg_pcg64* rng, int32_t flags,
                    void* stream, vpg_graph** out) {
  return vpg_graph_build_wait(rec, cluster_size, rng, flags, stream, nullptr, out);
}

int vpg_graph_info_get(const vpg_graph* g, vpg_graph_info* out) {
  return guarded([&] {
    g->sync_totals();
    *out = g->info;
  });
}

int vpg_graph_set_records(vpg_graph* g, const vpg_records* rec) {
  return guarded([&] {
    VPG_REQUIRE(rec->n == g->rec.n, VPG_EINVAL, "records of another size");
    g->rec = *rec;
  });
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

int vpg_graph_build_local(const vpg_records* rec, int64_t n_clusters, const int32_t* cl_size,
                          const int32_t* parent, const uint8_t* has_child, int64_t n_halo,
                          const double* halo_ipt, void* stream, vpg_graph** out) {
  *out = nullptr;
  vpg_graph* g = new vpg_graph();
  const int rc = guarded([&] {
    g->stream = as_stream(stream);
    g->rec = *rec;
    vpg::build_local(g, *rec, n_clusters, cl_size, parent, has_child, n_halo, halo_ipt, g->stream);
  });
  if (rc != VPG_OK) {
    delete g;
    return rc;
  }
  *out = g;
  return VPG_OK;
}

int vpg_graph_views_get(const vpg_graph* g, vpg_graph_views* v) {
  return guarded([&] {
    *v = vpg_graph_views{};
    v->n = g->n;
    v->m = g->m;
    v->n_halo = g->n_halo;
    v->perm = g->perm.get();
    v->clpos = g->clpos.get();
    vpg::ensure_cluster_ids(g, as_stream(nullptr));
    v->cluster_id = g->cluster_id.get();
    v->cl_off = g->cl_off.get();
    v->cl_size = g->cl_size.get();
    v->cl_center = g->cl_center.get();
    v->ref_of = g->ref_of.get();
    v->internal_of = g->internal_of.get();
    v->i0 = reinterpret_cast<float*>(g->i0.get());
    v->ibuf[0] = reinterpret_cast<float*>(g->ibuf[0].get());
    v->ibuf[1] = reinterpret_cast<float*>(g->ibuf[1].get());
    v->acc[0] = reinterpret_cast<float*>(g->acc[0].get());
    v->acc[1] = reinterpret_cast<float*>(g->acc[1].get());
    v->dbar = reinterpret_cast<float*>(g->dbar.get());
    v->term_max = g->term_max.get();
    v->red = g->red.get();
    v->ctl = g->ctl.get();
    v->performed = g->performed;
  });
}

int vpg_solve_begin(vpg_graph* g, int32_t iterations, double tol, void* stream) {
  return guarded([&] { vpg::solve_begin(g, g->rec, iterations, tol, as_stream(stream)); });
}

int vpg_solve_step(vpg_graph* g, int32_t t, void* stream) {
  return guarded([&] { vpg::solve_step(g, t, as_stream(stream)); });
}

int vpg_solve_control(vpg_graph* g, int32_t t, void* stream) {
  return guarded([&] { vpg::solve_control(g, t, as_stream(stream)); });
}

int vpg_solve_end(vpg_graph* g, double* residuals, int32_t* performed, void* stream) {
  return guarded([&] { vpg::solve_end(g, residuals, performed, false, as_stream(stream)); });
}

int vpg_splat_arrays(const vpg_paths* paths, const double* coeff, const int32_t* clpos,
                     const float* acc4, const float* dbar4, int64_t n_pixels, int32_t spp,
                     int32_t direct_mode, double* image, void* stream) {
  return guarded([&] {
    vpg::splat_arrays(*paths, coeff, clpos, reinterpret_cast<const float4*>(acc4),
                      reinterpret_cast<const float4*>(dbar4), n_pixels, spp, direct_mode, image,
                      as_stream(stream));
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

int vpg_trace_capture(const vpg_scene* scene, const vpg_trace_cfg* cfg, double* scratch,
                      int64_t capacity, uint64_t* counter, int64_t* counts, const vpg_paths* paths,
                      void* stream) {
  return guarded([&] {
    vpg::trace_capture(*scene, *cfg, scratch, capacity,
                       reinterpret_cast<unsigned long long*>(counter), counts, *paths,
                       as_stream(stream));
  });
}

int vpg_scatter_records(const double* scratch, int64_t n, const int64_t* rec_start,
                        int64_t path_begin, const vpg_records* out, void* stream) {
  return guarded([&] {
    vpg::scatter_records(scratch, n, rec_start, path_begin, *out, as_stream(stream));
  });
}

int vpg_extra_direct(const vpg_scene* scene, const vpg_records* rec, const vpg_paths* paths,
                     int64_t seed, int32_t n_extra, void* stream) {
  return guarded([&] { vpg::extra_direct(*scene, *rec, *paths, seed, n_extra, as_stream(stream)); });
}

int vpg_release_cached(void) {
  return guarded([&] { vpg::release_cached(); });
}

int vpg_extra_direct_range(const vpg_scene* scene, const vpg_records* rec, const vpg_paths* paths,
                           int64_t path_begin, int64_t seed, int32_t n_extra, void* stream) {
  return guarded([&] {
    vpg::extra_direct(*scene, *rec, *paths, seed, n_extra, as_stream(stream), path_begin);
  });
}

int vpg_reconstruct_paths(const vpg_records* rec, const vpg_paths* paths, const int64_t* path_ids,
                          int64_t count, double* estimate, double* max_ipt_diff, void* stream) {
  return guarded([&] {
    vpg::reconstruct_paths(*rec, *paths, path_ids, count, estimate, max_ipt_diff, as_stream(stream));
  });
}

}  // extern "C"

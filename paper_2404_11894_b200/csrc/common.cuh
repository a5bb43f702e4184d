// Shared runtime pieces of libvolpg_b200: error state, launch accounting,
// stream-ordered scratch allocation.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/volpg_b200.h"

namespace vpg {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

void set_last_error(const std::string& msg);
void count_launch(uint64_t n = 1);
void count_transfer(uint64_t h2d, uint64_t d2h);

// Optional per-kernel device timing (vpg_profile_*): CUDA events recorded on
// the launching stream around each launch, aggregated by kernel name.
bool profiling();
int prof_begin(const char* name, cudaStream_t s);
void prof_end(int token, cudaStream_t s);

#define VPG_CUDA(expr)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      throw ::vpg::Error(VPG_ECUDA, std::string(#expr " failed: ") + cudaGetErrorString(_e) + \
                                        " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

#define VPG_REQUIRE(cond, code, msg)                 \
  do {                                               \
    if (!(cond)) throw ::vpg::Error((code), (msg));  \
  } while (0)

// Device-side bounds checks, compiled in only for the checked build
// (python tools/build_variant.py checked -DVPG_CHECKED, then the GPU tests
// with VPG_LIB_VARIANT=checked): compute-sanitizer is not available on the
// GPU pool, so the kernels assert their own index ranges there.  A failed
// check prints the condition and traps (the test's launch then errors).
#ifdef VPG_CHECKED
#define VPG_CHECK(cond)                                                                    \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("VPG_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             int(blockIdx.x), int(threadIdx.x));                                          \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define VPG_CHECK(cond) \
  do {                  \
  } while (0)
#endif

// Launch wrapper: counts the launch and surfaces configuration errors.
#define VPG_LAUNCH(kernel, grid, block, smem, stream, ...)                 \
  do {                                                                     \
    if ((grid) > 0) {                                                      \
      const int _tok = ::vpg::profiling() ? ::vpg::prof_begin(#kernel, stream) : -1; \
      kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);          \
      if (_tok >= 0) ::vpg::prof_end(_tok, stream);                        \
      ::vpg::count_launch();                                               \
      VPG_CUDA(cudaGetLastError());                                        \
    }                                                                      \
  } while (0)

// Run `body`, translating exceptions into the C ABI's error codes.
template <class F>
int guarded(F&& body) {
  try {
    body();
    return VPG_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return VPG_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return VPG_ECUDA;
  }
}

// ------------------------------------------------------ device scratch
// Stream-ordered allocation from the device's default memory pool; the pool
// keeps freed blocks (release threshold raised once), so repeated builds of
// the same size do not return to the driver.
void* dalloc(size_t bytes, cudaStream_t s);
void dfree(void* p, cudaStream_t s);

template <class T>
struct DBuf {
  T* ptr = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(size_t count, cudaStream_t stream) { alloc(count, stream); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : ptr(o.ptr), n(o.n), s(o.s) { o.ptr = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); ptr = o.ptr; n = o.n; s = o.s; o.ptr = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count, cudaStream_t stream) {
    release();
    s = stream;
    n = count;
    ptr = static_cast<T*>(dalloc(count * sizeof(T) + 16, stream));
  }
  void release() {
    if (ptr) dfree(ptr, s);
    ptr = nullptr;
    n = 0;
  }
  T* get() const { return ptr; }
  size_t bytes() const { return n * sizeof(T); }
};

// Persistent device scratch for large build temporaries, keyed by (stream,
// tag): grown with cudaMalloc when a larger size is requested, never returned
// to the pool, so steady-state builds allocate nothing.  Calls on one stream
// are ordered, so reuse across successive builds on that stream is safe.
void* scratch(cudaStream_t s, const char* tag, size_t bytes);

template <class T>
T* scratch_of(cudaStream_t s, const char* tag, size_t count) {
  return static_cast<T*>(scratch(s, tag, count * sizeof(T) + 16));
}

// Page-locked host staging (cudaMallocHost), recycled through a process-wide
// cache so repeated builds do not pay for pinning.
void* halloc(size_t bytes);
void hfree(void* p, size_t bytes);

template <class T>
struct HostBuf {
  T* ptr = nullptr;
  size_t n = 0;
  HostBuf() = default;
  explicit HostBuf(size_t count) { alloc(count); }
  HostBuf(const HostBuf&) = delete;
  HostBuf& operator=(const HostBuf&) = delete;
  ~HostBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    ptr = static_cast<T*>(halloc(count * sizeof(T) + 16));
  }
  void release() {
    if (ptr) hfree(ptr, n * sizeof(T) + 16);
    ptr = nullptr;
    n = 0;
  }
  T* get() const { return ptr; }
  T& operator[](size_t i) const { return ptr[i]; }
};

inline int grid_for(int64_t work, int block, int max_blocks = 148 * 16) {
  int64_t g = (work + block - 1) / block;
  if (g > max_blocks) g = max_blocks;
  return int(g);
}

int sm_count();
// free the scratch buffers and trim the allocation pool (vpg_release_cached)
void release_cached();
// cudaFuncAttributeMaxDynamicSharedMemorySize, raised once per (device, kernel)
void ensure_dynamic_smem(const void* func, size_t bytes);

}  // namespace vpg

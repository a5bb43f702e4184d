// Path-graph clustering on the device, bit-exact with the reference.
//
// Reference: pathgraph/clustering.py:28-148 (+ graph.py:59-60 for the class
// keys and RNG).  Per compatibility class (ascending key kind<<32|class_id):
//   1. host: m = ceil(n/K) centers = Generator.choice(n, m)          (:51)
//   2. device: uniform grid with the reference's lo/cell (:102-106); centers
//      radix-sorted by cell key into an open-addressing cell table; one
//      thread per point scans the 27-cell neighbourhood with fp64 distances
//      rounded like numpy ((dx*dx+dy*dy)+dz*dz, no FMA) and lowest-center
//      ties (:121-137)
//   3. device: points with an empty neighbourhood or best >= cell fall back to
//      the exact global argmin (:129-131,138-147), one warp per point
//   4. device: stable radix sort (center, record) = groups in ascending record
//      order (:55)
//   5. host: LIFO split loop over groups > 2K (:58-85) with the same RNG
//   6. device: clusters numbered in group order, skipping empty groups,
//      continuing across classes (:87-93); cluster-major permutation.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <functional>
#include <thread>
#include <vector>

#include "graph.cuh"
#include "host_rng.hpp"

namespace vpg {
namespace {

constexpr uint64_t kEmpty = 0xFFFFFFFFFFFFFFFFull;
constexpr int kMaxClasses = 256;
constexpr int kSlotsPerKind = 65536;

struct CellEntry {
  unsigned long long key;
  int32_t start, end;
};

// order-preserving unsigned encoding of a double (for atomic min/max)
__host__ __device__ inline uint64_t order_key(double x) {
#ifdef __CUDA_ARCH__
  uint64_t b = uint64_t(__double_as_longlong(x));
#else
  uint64_t b;
  memcpy(&b, &x, 8);
#endif
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
inline double order_key_inv(uint64_t k) {
  uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  double x;
  memcpy(&x, &b, 8);
  return x;
}

__device__ __forceinline__ double dist2_exact(double ax, double ay, double az, double bx,
                                              double by, double bz) {
  const double dx = __dsub_rn(ax, bx), dy = __dsub_rn(ay, by), dz = __dsub_rn(az, bz);
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

__device__ __forceinline__ long long cell_coord(double p, double lo, double cell) {
  return (long long)floor(__ddiv_rn(__dsub_rn(p, lo), cell));
}

__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct GridParams {
  double lo[3];
  double cell;
  double slack;        // bound on fp error of a cell index, in cells
  long long dims[3];   // cells per axis covering the class bounding box
  long long max_dim;
  int packed;  // 1: key = packed (x+1,y+1,z+1) in 21 bits each; 0: hashed triple
  int m;       // centers in this class
  uint64_t table_mask;
};

__device__ __forceinline__ uint64_t cell_key(const GridParams& gp, long long x, long long y,
                                             long long z) {
  if (gp.packed)  // dense index over the grid padded by two cells per side
    return (uint64_t(x + 2) * uint64_t(gp.dims[1] + 4) + uint64_t(y + 2)) * uint64_t(gp.dims[2] + 4) +
           uint64_t(z + 2);
  uint64_t h = mix64(uint64_t(x) * 0x9E3779B97F4A7C15ull ^ mix64(uint64_t(y) + 0x632BE59BD9B4E019ull) ^
                     mix64(uint64_t(z) * 0xD1342543DE82EF95ull + 7));
  return h & 0x7FFFFFFFFFFFFFFFull;
}

__device__ __forceinline__ uint64_t table_slot(uint64_t key, uint64_t mask) {
  return mix64(key) & mask;
}

// ------------------------------------------------------------ kernels

__global__ void k_class_bitmap(const uint8_t* __restrict__ kind, const int32_t* __restrict__ cls,
                               int64_t n, uint32_t* bitmap, int32_t* err) {
  // a thread sets a class's bit only when its slot differs from the last
  // one it saw, and only while the bit is still clear (the few classes would
  // otherwise serialise every warp on one word)
  uint32_t last = ~0u;
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int k = kind[r];
    const int c = cls[r];
    if (k > 1 || c < 0 || c >= kSlotsPerKind) {
      atomicExch(err, 1);
      continue;
    }
    const uint32_t slot = uint32_t(k * kSlotsPerKind + c);
    if (slot == last) continue;
    last = slot;
    const uint32_t bit = 1u << (slot & 31);
    if (!(*reinterpret_cast<volatile uint32_t*>(&bitmap[slot >> 5]) & bit))
      atomicOr(&bitmap[slot >> 5], bit);
  }
}

// Per-class counts and position bounds; also the class index of each record.
__global__ void k_class_stats(const uint8_t* __restrict__ kind, const int32_t* __restrict__ cls,
                              const double* __restrict__ pos, int64_t n,
                              const uint32_t* __restrict__ slots, int n_cls,
                              uint8_t* __restrict__ cls_idx, unsigned long long* counts,
                              unsigned long long* mins, unsigned long long* maxs) {
  __shared__ uint32_t s_slots[kMaxClasses];
  __shared__ unsigned long long s_cnt[kMaxClasses], s_mn[kMaxClasses * 3], s_mx[kMaxClasses * 3];
  for (int i = threadIdx.x; i < n_cls; i += blockDim.x) {
    s_slots[i] = slots[i];
    s_cnt[i] = 0;
    for (int a = 0; a < 3; ++a) {
      s_mn[i * 3 + a] = ~0ull;
      s_mx[i * 3 + a] = 0ull;
    }
  }
  __syncthreads();
  int cur = -1;
  unsigned long long cnt = 0, mn[3] = {~0ull, ~0ull, ~0ull}, mx[3] = {0, 0, 0};
  auto flush = [&]() {
    if (cur < 0 || cnt == 0) return;
    atomicAdd(&s_cnt[cur], cnt);
    for (int a = 0; a < 3; ++a) {
      atomicMin(&s_mn[cur * 3 + a], mn[a]);
      atomicMax(&s_mx[cur * 3 + a], mx[a]);
      mn[a] = ~0ull;
      mx[a] = 0;
    }
    cnt = 0;
  };
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t slot = uint32_t(kind[r]) * kSlotsPerKind + uint32_t(cls[r]);
    int lo = 0, hi = n_cls - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (s_slots[mid] < slot) lo = mid + 1; else hi = mid;
    }
    if (lo != cur) {
      flush();
      cur = lo;
    }
    if (cls_idx) cls_idx[r] = uint8_t(lo);
    ++cnt;
    for (int a = 0; a < 3; ++a) {
      const uint64_t k = order_key(pos[r * 3 + a]);
      mn[a] = mn[a] < k ? mn[a] : k;
      mx[a] = mx[a] > k ? mx[a] : k;
    }
  }
  flush();
  __syncthreads();
  for (int i = threadIdx.x; i < n_cls; i += blockDim.x) {
    if (s_cnt[i] == 0) continue;
    atomicAdd(&counts[i], s_cnt[i]);
    for (int a = 0; a < 3; ++a) {
      atomicMin(&mins[i * 3 + a], s_mn[i * 3 + a]);
      atomicMax(&maxs[i * 3 + a], s_mx[i * 3 + a]);
    }
  }
}

__global__ void k_iota(int32_t* out, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = int32_t(i);
}

__device__ __forceinline__ int64_t class_row(const int32_t* rows, int64_t row_off, int64_t i) {
  return rows ? int64_t(rows[row_off + i]) : row_off + i;
}

// Center positions, record ids and cell keys.
__global__ void k_center_setup(const int32_t* __restrict__ local, int m, const int32_t* rows,
                               int64_t row_off, const double* __restrict__ pos, GridParams gp,
                               double* __restrict__ cpos, int32_t* __restrict__ crec,
                               unsigned long long* __restrict__ keys, int32_t* __restrict__ ids) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
    const int64_t r = class_row(rows, row_off, local[j]);
    const double x = pos[r * 3], y = pos[r * 3 + 1], z = pos[r * 3 + 2];
    cpos[j * 3] = x;
    cpos[j * 3 + 1] = y;
    cpos[j * 3 + 2] = z;
    crec[j] = int32_t(r);
    keys[j] = cell_key(gp, cell_coord(x, gp.lo[0], gp.cell), cell_coord(y, gp.lo[1], gp.cell),
                       cell_coord(z, gp.lo[2], gp.cell));
    ids[j] = j;
  }
}

// Cell keys of given centers (assign_nearest).
__global__ void k_center_keys(const double* __restrict__ cpos, int m, GridParams gp,
                              unsigned long long* __restrict__ keys, int32_t* __restrict__ ids) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
    keys[j] = cell_key(gp, cell_coord(cpos[j * 3], gp.lo[0], gp.cell),
                       cell_coord(cpos[j * 3 + 1], gp.lo[1], gp.cell),
                       cell_coord(cpos[j * 3 + 2], gp.lo[2], gp.cell));
    ids[j] = j;
  }
}

// Sorted centers -> packed positions; run heads inserted into the cell table.
__global__ void k_center_table(const unsigned long long* __restrict__ skeys,
                               const int32_t* __restrict__ sids, const double* __restrict__ cpos,
                               int m, GridParams gp, double4* __restrict__ spos,
                               CellEntry* table) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int j = sids[i];
    spos[i] = make_double4(cpos[j * 3], cpos[j * 3 + 1], cpos[j * 3 + 2], __longlong_as_double((long long)j));
    const unsigned long long key = skeys[i];
    if (table && (i == 0 || skeys[i - 1] != key)) {
      uint64_t slot = table_slot(key, gp.table_mask);
      while (true) {
        const unsigned long long prev = atomicCAS(&table[slot].key, kEmpty, key);
        if (prev == kEmpty) {
          table[slot].start = i;
          break;
        }
        slot = (slot + 1) & gp.table_mask;
      }
    }
  }
}

__device__ __forceinline__ const CellEntry* table_find(const CellEntry* table, uint64_t key,
                                                       uint64_t mask) {
  uint64_t slot = table_slot(key, mask);
  while (true) {
    const CellEntry* e = &table[slot];
    const unsigned long long k = e->key;
    if (k == key) return e;
    if (k == kEmpty) return nullptr;
    slot = (slot + 1) & mask;
  }
}

// Cell -> [first, end) of its centers among the key-sorted centers: a direct
// array over the dense packed keys when the grid is small enough (one load),
// else the hash table.
struct CellIndex {
  const CellEntry* hash;
  const int2* dense;
  uint64_t mask;
  __device__ __forceinline__ bool find(uint64_t key, int& start, int& end) const {
    if (dense) {
      const int2 e = dense[key];
      start = e.x;
      end = e.y;
      return e.y > e.x;
    }
    const CellEntry* e = table_find(hash, key, mask);
    if (!e) return false;
    start = e->start;
    end = e->end;
    return true;
  }
};

__global__ void k_center_dense(const unsigned long long* __restrict__ skeys, int m,
                               int2* __restrict__ dense) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const unsigned long long key = skeys[i];
    if (i == 0 || skeys[i - 1] != key) dense[key].x = i;
    if (i == m - 1 || skeys[i + 1] != key) dense[key].y = i + 1;
  }
}

__global__ void k_center_table_ends(const unsigned long long* __restrict__ skeys, int m,
                                    GridParams gp, CellEntry* table) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const unsigned long long key = skeys[i];
    if (i == m - 1 || skeys[i + 1] != key) {
      CellEntry* e = const_cast<CellEntry*>(table_find(table, key, gp.table_mask));
      e->end = i + 1;
    }
  }
}

struct Best {
  double d2;
  int j;
};
// a point sent on to the exact fallback, with its best over the 27 cells
struct FbEntry {
  double d2;
  int32_t i, j;
};
__device__ __forceinline__ void best_update(Best& b, double d2, int j) {
  if (d2 < b.d2 || (d2 == b.d2 && j < b.j)) {
    b.d2 = d2;
    b.j = j;
  }
}

// Scan the centers of one cell (key) into `b`.
__device__ __forceinline__ void scan_cell(const GridParams& gp, const CellIndex& table,
                                          const double4* __restrict__ spos, long long cx,
                                          long long cy, long long cz, double px, double py,
                                          double pz, Best& b) {
  int start, end;
  if (!table.find(cell_key(gp, cx, cy, cz), start, end)) return;
  for (int t = start; t < end; ++t) {
    const double4 c = spos[t];
    if (!gp.packed) {  // hashed keys: confirm the cell really matches
      if (cell_coord(c.x, gp.lo[0], gp.cell) != cx || cell_coord(c.y, gp.lo[1], gp.cell) != cy ||
          cell_coord(c.z, gp.lo[2], gp.cell) != cz)
        continue;
    }
    best_update(b, dist2_exact(px, py, pz, c.x, c.y, c.z), int(__double_as_longlong(c.w)));
  }
}


// Z-order key of each center's cell: part A's clusters are laid out in this
// order (any order is valid; ref_of keeps the reference numbering) so that
// spatially close clusters -- and the continuation parents a row scatters
// into during the solve -- are close in memory.
__device__ __forceinline__ unsigned long long spread3(unsigned long long v) {
  v &= 0x1FFFFFull;
  v = (v | (v << 32)) & 0x1F00000000FFFFull;
  v = (v | (v << 16)) & 0x1F0000FF0000FFull;
  v = (v | (v << 8)) & 0x100F00F00F00F00Full;
  v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

__global__ void k_center_morton(const double* __restrict__ cpos, int m, GridParams gp,
                                unsigned long long* __restrict__ keys, int32_t* __restrict__ ids) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
    unsigned long long c[3];
    for (int a = 0; a < 3; ++a) {
      const long long v = cell_coord(cpos[j * 3 + a], gp.lo[a], gp.cell);
      c[a] = (unsigned long long)(v < 0 ? 0 : (v > 0x1FFFFF ? 0x1FFFFF : v));
    }
    keys[j] = spread3(c[0]) | (spread3(c[1]) << 1) | (spread3(c[2]) << 2);
    ids[j] = j;
  }
}

// ------------------------------------ Generator.choice tail shuffle on device
// numpy's partial Fisher-Yates (n > 10000, m > n // 50): step k swaps
// positions i_k = n-1-k and j_k (drawn on the host).  Position i_k is final
// after step k, so out[m-1-k] = value at j_k before step k, and step k writes
// the value of position i_k into j_k.  With the (j, k) pairs sorted, the
// previous writer of any position is found by search, and values follow short
// chains of earlier writers back to an untouched position.
__global__ void k_swap_keys(const int32_t* __restrict__ target, int64_t steps,
                            unsigned long long* __restrict__ keys) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < steps;
       k += int64_t(gridDim.x) * blockDim.x)
    keys[k] = (unsigned long long)(uint32_t(target[k])) << 32 | uint32_t(k);
}

// Largest step k' < k that wrote position p, or -1.
__device__ __forceinline__ int64_t last_writer(const unsigned long long* __restrict__ sk,
                                               int64_t steps, uint32_t p, int64_t k) {
  const unsigned long long key = (unsigned long long)p << 32 | uint32_t(k);
  int64_t lo = 0, hi = steps;  // first index with sk >= key
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (sk[mid] < key) lo = mid + 1; else hi = mid;
  }
  if (lo == 0) return -1;
  const unsigned long long prev = sk[lo - 1];
  return uint32_t(prev >> 32) == p ? int64_t(uint32_t(prev)) : -1;
}

// prev_i[k]: last writer of position i_k before step k.
__global__ void k_swap_links(const unsigned long long* __restrict__ sk, int64_t steps, int64_t n,
                             int32_t* __restrict__ prev_i) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < steps;
       k += int64_t(gridDim.x) * blockDim.x)
    prev_i[k] = int32_t(last_writer(sk, steps, uint32_t(n - 1 - k), k));
}

// value written by step k = the untouched position at the end of its chain
__device__ __forceinline__ int32_t written_value(const int32_t* __restrict__ prev_i, int64_t n,
                                                 int64_t k) {
  while (prev_i[k] >= 0) k = prev_i[k];
  return int32_t(n - 1 - k);
}

__global__ void k_swap_resolve(const int32_t* __restrict__ target,
                               const unsigned long long* __restrict__ sk,
                               const int32_t* __restrict__ prev_i, int64_t steps, int64_t n,
                               int64_t m, int32_t* __restrict__ out) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < steps;
       k += int64_t(gridDim.x) * blockDim.x) {
    const int32_t j = target[k];
    const int64_t w = last_writer(sk, steps, uint32_t(j), k);
    out[m - 1 - k] = w < 0 ? j : written_value(prev_i, n, w);
  }
  // m == n: position 0 is never a swap source; its final value
  if (blockIdx.x == 0 && threadIdx.x == 0 && n == m) {
    const int64_t w = last_writer(sk, steps, 0u, steps);
    out[0] = w < 0 ? 0 : written_value(prev_i, n, w);
  }
}

// ------------------------------------------------ cell-sorted assignment
constexpr long long kShellBudget = 4096;  // cells one fallback point may enumerate
constexpr int kAssignWarps = 8;

// Sort key of a point's cell: the cell key (dense over the padded grid when
// packed, else hashed: ties only cost extra candidates).
__device__ __forceinline__ unsigned long long sort_key(const GridParams& gp, long long x,
                                                       long long y, long long z) {
  return cell_key(gp, x, y, z);
}

__global__ void k_point_keys(const int32_t* rows, int64_t row_off, int64_t n,
                             const double* __restrict__ pos, GridParams gp,
                             unsigned long long* __restrict__ keys, int32_t* __restrict__ ids) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = class_row(rows, row_off, i);
    keys[i] = sort_key(gp, cell_coord(pos[r * 3], gp.lo[0], gp.cell),
                       cell_coord(pos[r * 3 + 1], gp.lo[1], gp.cell),
                       cell_coord(pos[r * 3 + 2], gp.lo[2], gp.cell));
    ids[i] = int32_t(i);
  }
}

// Counting sort of the points by cell (dense packed keys): count, scan,
// scatter.  Points of one cell land in arbitrary order, which the assignment
// does not see (each point's nearest center is exact on its own).
constexpr int kOctShift = 29;  // octant bits in the cell-sorted point ids

// Also the point's octant in its cell (bit a: the upper half along axis a),
// carried into cell order for the assignment's batches.
__device__ __forceinline__ int cell_and_octant(double p, double lo, double cell, long long& c) {
  const double t = __ddiv_rn(__dsub_rn(p, lo), cell);
  c = (long long)floor(t);
  return int((long long)floor(2.0 * t) & 1);  // 2t is exact
}

__global__ void k_cell_count(const int32_t* rows, int64_t row_off, int64_t n,
                             const double* __restrict__ pos, GridParams gp,
                             int32_t* __restrict__ counts, int32_t* __restrict__ pkey,
                             uint8_t* __restrict__ poct) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = class_row(rows, row_off, i);
    long long x, y, z;
    const int o = cell_and_octant(pos[r * 3], gp.lo[0], gp.cell, x) |
                  (cell_and_octant(pos[r * 3 + 1], gp.lo[1], gp.cell, y) << 1) |
                  (cell_and_octant(pos[r * 3 + 2], gp.lo[2], gp.cell, z) << 2);
    const int32_t key = int32_t(cell_key(gp, x, y, z));
    pkey[i] = key;
    if (poct) poct[i] = uint8_t(o);
    atomicAdd(&counts[key], 1);
  }
}

// poct (n < 2^29): the octant rides in bits 29..31 of the sorted ids
__global__ void k_cell_scatter(int64_t n, const int32_t* __restrict__ pkey,
                               const uint8_t* __restrict__ poct, const int32_t* __restrict__ offs,
                               int32_t* __restrict__ counts, int32_t* __restrict__ sorted_ids) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t key = pkey[i];
    const int32_t at = offs[key] + atomicSub(&counts[key], 1) - 1;
    sorted_ids[at] = int32_t(uint32_t(i) | (poct ? uint32_t(poct[i]) << kOctShift : 0u));
  }
}

struct CellNonEmpty {
  const int32_t* offs;
  __host__ __device__ bool operator()(int32_t c) const { return offs[c + 1] > offs[c]; }
};

__global__ void k_cell_runs(const int32_t* __restrict__ cells, const int32_t* __restrict__ n_sel,
                            const int32_t* __restrict__ offs, int32_t* __restrict__ run_start,
                            int32_t* __restrict__ run_len) {
  const int n = *n_sel;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int32_t c = cells[i];
    run_start[i] = offs[c];
    run_len[i] = offs[c + 1] - offs[c];
  }
}

// Neighbour cell v of the visit order (k = 9 dx + 3 dy + dz, offsets d - 1):
// the home cell, the 6 faces, then the 12 edges and the 8 corners.
__host__ __device__ constexpr int visit_cell(int v) {
  switch (v) {
    case 0: return 13;
    case 1: return 4;   case 2: return 10;  case 3: return 12;  case 4: return 14;
    case 5: return 16;  case 6: return 22;
    case 7: return 1;   case 8: return 3;   case 9: return 5;   case 10: return 7;
    case 11: return 9;  case 12: return 11; case 13: return 15; case 14: return 17;
    case 15: return 19; case 16: return 21; case 17: return 23; case 18: return 25;
    case 19: return 0;  case 20: return 2;  case 21: return 6;  case 22: return 8;
    case 23: return 18; case 24: return 20; case 25: return 24; default: return 26;
  }
}
// the same order for runtime indices
#define VPG_V(i) uint8_t(visit_cell(i))
__constant__ uint8_t kVisitOrder[27] = {
    VPG_V(0),  VPG_V(1),  VPG_V(2),  VPG_V(3),  VPG_V(4),  VPG_V(5),  VPG_V(6),
    VPG_V(7),  VPG_V(8),  VPG_V(9),  VPG_V(10), VPG_V(11), VPG_V(12), VPG_V(13),
    VPG_V(14), VPG_V(15), VPG_V(16), VPG_V(17), VPG_V(18), VPG_V(19), VPG_V(20),
    VPG_V(21), VPG_V(22), VPG_V(23), VPG_V(24), VPG_V(25), VPG_V(26)};
#undef VPG_V
constexpr int kNearCells = 7;   // home + faces: always scanned
#ifndef VPG_ASSIGN_CAND
#define VPG_ASSIGN_CAND 240
#endif
#ifndef VPG_ASSIGN_RUN
#define VPG_ASSIGN_RUN 256
#endif
#ifndef VPG_ASSIGN_MINB
#define VPG_ASSIGN_MINB 3
#endif
constexpr int kCandCap = VPG_ASSIGN_CAND;  // candidate centers staged per warp
constexpr int kRunCap = VPG_ASSIGN_RUN;    // points put in octant order at a time

// (out of line: only hashed grids need it, and three inlined divisions per
// call site would bloat the assignment loop out of the instruction cache)
__device__ __noinline__ bool center_in_cell(double cx, double cy, double cz, const GridParams& gp,
                                            long long x, long long y, long long z) {
  return cell_coord(cx, gp.lo[0], gp.cell) == x && cell_coord(cy, gp.lo[1], gp.cell) == y &&
         cell_coord(cz, gp.lo[2], gp.cell) == z;
}

__device__ __forceinline__ int octant_of(double x, double y, double z, const GridParams& gp,
                                         long long cx, long long cy, long long cz,
                                         double inv_cell) {
  return int((x - gp.lo[0]) * inv_cell - double(cx) >= 0.5) |
         (int((y - gp.lo[1]) * inv_cell - double(cy) >= 0.5) << 1) |
         (int((z - gp.lo[2]) * inv_cell - double(cz) >= 0.5) << 2);
}

// One warp per run of points sharing a cell (points sorted by cell): lanes
// 0..26 look up the 27 neighbour cells once, in visit order -- exactly the
// reference's per-cell candidate list (clustering.py:121-137).  The run's
// points are taken kRunCap at a time in octant order, then 32 at a time scan
// the home cell and the faces, and of the 20 edge and corner cells only those
// some lane can still reach: a cell is skipped when, for every lane, the
// point's distance to the cell's box (in cell units, fp32, shrunk by a margin
// far above the rounding of the cell indices) exceeds its best squared
// distance so far, so all its centers are strictly farther and the
// lexicographic (d2, center) minimum over the 27 cells is unchanged.  Octant
// order makes the 32 points of a batch neighbours, so they skip the same
// cells.  The candidates are staged in shared memory once per run, or, for a
// crowded neighbourhood (more than kCandCap), cell by cell for each batch.
__global__ void __launch_bounds__(kAssignWarps * 32, VPG_ASSIGN_MINB)
k_assign_cells(const int32_t* rows, int64_t row_off, const double* __restrict__ pos, GridParams gp,
               CellIndex table, const double4* __restrict__ spos,
               const int32_t* __restrict__ sorted_ids, int oct_in_ids,
               const int32_t* __restrict__ run_start, const int32_t* __restrict__ run_len,
               const int32_t* __restrict__ n_runs, int32_t* __restrict__ assign,
               FbEntry* __restrict__ fb_list, int32_t* __restrict__ fb_count) {
  constexpr unsigned kFull = 0xFFFFFFFFu;
  constexpr float kMargin = 1e-4f;  // cells
  extern __shared__ __align__(16) unsigned char assign_smem[];
  double4* cand = reinterpret_cast<double4*>(assign_smem) + (threadIdx.x >> 5) * kCandCap;
  int32_t* run_ids = reinterpret_cast<int32_t*>(assign_smem + sizeof(double4) * kCandCap *
                                                                  kAssignWarps) +
                     (threadIdx.x >> 5) * kRunCap;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int runs = *n_runs;
  const int warps = gridDim.x * kAssignWarps;
  const double inv_cell = 1.0 / gp.cell;
  const double inv_cell2 = inv_cell * inv_cell;
  for (int run = blockIdx.x * kAssignWarps + wid; run < runs; run += warps) {
    const int32_t b = run_start[run], len = run_len[run];
    const uint32_t id_mask = oct_in_ids ? (1u << kOctShift) - 1u : 0xFFFFFFFFu;
    const int64_t r0 = class_row(rows, row_off, int32_t(sorted_ids[b] & id_mask));
    const long long cx = cell_coord(pos[r0 * 3], gp.lo[0], gp.cell);
    const long long cy = cell_coord(pos[r0 * 3 + 1], gp.lo[1], gp.cell);
    const long long cz = cell_coord(pos[r0 * 3 + 2], gp.lo[2], gp.cell);
    int c_start = 0, c_cnt = 0;
    if (lane < 27) {
      const int k = visit_cell(lane);
      int st, en;
      if (table.find(cell_key(gp, cx + k / 9 - 1, cy + (k / 3) % 3 - 1, cz + k % 3 - 1), st, en)) {
        c_start = st;
        c_cnt = en - st;
      }
    }
    const unsigned nonempty = __ballot_sync(kFull, c_cnt > 0);
    int incl = c_cnt;  // inclusive warp scan of candidate counts (visit order)
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(kFull, incl, off);
      if (lane >= off) incl += v;
    }
    const int total = __shfl_sync(kFull, incl, 31);
    const bool staged = total <= kCandCap;
    // copy candidates [i0, i0 + cnt) of the visit order into cand[0 ..):
    // index idx is in visit cell v = #lanes whose inclusive count is <= idx;
    // with hashed keys a colliding cell's centers become +inf
    auto stage = [&](int i0, int cnt) {
#pragma unroll 1
      for (int t0 = 0; t0 < cnt; t0 += 32) {  // warp-uniform: the shuffles need every lane
        const int t = t0 + lane;
        const int idx = i0 + t;
        int v = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const int c = __shfl_sync(kFull, incl, v + step - 1);
          if (c <= idx) v += step;
        }
        const int first = __shfl_sync(kFull, incl - c_cnt, v);
        const int from = __shfl_sync(kFull, c_start, v) + (idx - first);
        if (t >= cnt) continue;
        VPG_CHECK(t < kCandCap && v < 27 && from >= 0);
        double4 c = spos[from];
        if (!gp.packed) {
          const int k = kVisitOrder[v];
          if (!center_in_cell(c.x, c.y, c.z, gp, cx + k / 9 - 1, cy + (k / 3) % 3 - 1,
                              cz + k % 3 - 1))
            c = make_double4(INFINITY, INFINITY, INFINITY, __longlong_as_double(0x7FFFFFFFLL));
        }
        cand[t] = c;
      }
    };
    if (staged) {
      stage(0, total);
      __syncwarp();
    }
    const int c_first = incl - c_cnt;  // visit-order offset of each cell
#pragma unroll 1
    for (int s0 = 0; s0 < len; s0 += kRunCap) {
      const int seg = len - s0 < kRunCap ? len - s0 : kRunCap;
      // the segment's point ids into run_ids, octant by octant (a counting
      // sort; lanes 0..7 hold the octant counts, then their bases)
      int base = 0;
#pragma unroll 1
      for (int pass = 0; pass < 2; ++pass) {
#pragma unroll 1
        for (int c0 = 0; c0 < seg; c0 += 32) {
          int o = 8;
          int32_t id = 0;
          if (c0 + lane < seg) {
            id = sorted_ids[b + s0 + c0 + lane];
            if (oct_in_ids) {
              o = int(uint32_t(id) >> kOctShift);
              id = int32_t(uint32_t(id) & id_mask);
            } else {
              const int64_t r = class_row(rows, row_off, id);
              o = octant_of(pos[r * 3], pos[r * 3 + 1], pos[r * 3 + 2], gp, cx, cy, cz, inv_cell);
            }
          }
          if (pass == 1) {
            const unsigned peers = __match_any_sync(kFull, o);
            const int at = __shfl_sync(kFull, base, o & 7) + __popc(peers & ((1u << lane) - 1u));
            VPG_CHECK(o == 8 || (at >= 0 && at < seg));
            if (o < 8) run_ids[at] = id;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int cnt = __popc(__ballot_sync(kFull, o == q));
            if (lane == q) base += cnt;
          }
        }
        if (pass == 0) {
          const int hist = base;
          for (int off = 1; off < 8; off <<= 1) {
            const int v = __shfl_up_sync(kFull, base, off);
            if (lane >= off) base += v;
          }
          base -= hist;
        }
      }
      __syncwarp();
      // the next batch's point is loaded while this one scans
      int32_t ni = 0;
      double nx = 0.0, ny = 0.0, nz = 0.0;
      auto load_point = [&](int pb) {
        if (pb + lane < seg) {
          ni = run_ids[pb + lane];
          const int64_t r = class_row(rows, row_off, ni);
          nx = pos[r * 3];
          ny = pos[r * 3 + 1];
          nz = pos[r * 3 + 2];
        }
      };
      load_point(0);
#pragma unroll 1
      for (int pb = 0; pb < seg; pb += 32) {
        const bool active = pb + lane < seg;
        const int32_t i = ni;
        const double px = nx, py = ny, pz = nz;
        if (pb + 32 < seg) load_point(pb + 32);
        Best best{INFINITY, 0x7FFFFFFF};
        auto scan = [&](int q0, int cnt) {
#pragma unroll 4
          for (int q = q0; q < q0 + cnt; ++q) {
            const double4 c = cand[q];
            best_update(best, dist2_exact(px, py, pz, c.x, c.y, c.z),
                        int(__double_as_longlong(c.w)));
          }
        };
        // visit the cells whose bits are set: staged, or copied cell by cell
        // (crowded)
        auto visit = [&](unsigned cells) {
          while (cells) {
            const int v = __ffs(cells) - 1;
            cells &= cells - 1;
            const int kb = __shfl_sync(kFull, c_first, v), kc = __shfl_sync(kFull, c_cnt, v);
            if (staged) {
              VPG_CHECK(kb >= 0 && kb + kc <= total && total <= kCandCap);
              scan(kb, kc);
            } else {
              for (int t0 = 0; t0 < kc; t0 += kCandCap) {
                const int cnt = kc - t0 < kCandCap ? kc - t0 : kCandCap;
                __syncwarp();
                stage(kb + t0, cnt);
                __syncwarp();
                scan(0, cnt);
              }
            }
          }
        };
        // home cell and faces
        visit(nonempty & ((1u << kNearCells) - 1u));
        // edges and corners some lane can still reach
        unsigned need = 0;
        if (active) {
          float sq[3][2];
          const double t[3] = {(px - gp.lo[0]) * inv_cell - double(cx),
                               (py - gp.lo[1]) * inv_cell - double(cy),
                               (pz - gp.lo[2]) * inv_cell - double(cz)};
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const float lo_gap = fmaxf(float(t[a]) - kMargin, 0.f);
            const float hi_gap = fmaxf(float(1.0 - t[a]) - kMargin, 0.f);
            sq[a][0] = lo_gap * lo_gap;
            sq[a][1] = hi_gap * hi_gap;
          }
          const float reach = float(best.d2 * inv_cell2) * 1.0001f;
#pragma unroll
          for (int v = kNearCells; v < 27; ++v) {
            const int k = visit_cell(v);
            const int dx = k / 9, dy = (k / 3) % 3, dz = k % 3;
            float lb = 0.f;
            if (dx != 1) lb += sq[0][dx >> 1];
            if (dy != 1) lb += sq[1][dy >> 1];
            if (dz != 1) lb += sq[2][dz >> 1];
            if (!(lb > reach)) need |= 1u << v;
          }
        }
        visit(__reduce_or_sync(kFull, need) & nonempty);
        if (active) {
          if (best.j == 0x7FFFFFFF || !(__dsqrt_rn(best.d2) < gp.cell)) {
            fb_list[atomicAdd(fb_count, 1)] = FbEntry{best.d2, i, best.j};
            assign[i] = -1;
          } else {
            assign[i] = best.j;
          }
        }
      }
      __syncwarp();
    }
  }
}
constexpr size_t kAssignSmem = (sizeof(double4) * kCandCap + sizeof(int32_t) * kRunCap) *
                               kAssignWarps;

__device__ __forceinline__ void warp_best(Best& b) {
  for (int off = 16; off; off >>= 1) {
    const double od = __shfl_xor_sync(0xFFFFFFFFu, b.d2, off);
    const int oj = __shfl_xor_sync(0xFFFFFFFFu, b.j, off);
    best_update(b, od, oj);
  }
}

// Exact global argmin (ties -> lowest center) for the points the reference
// sends to its brute-force scan (clustering.py:129-147).  One warp per point
// grows Chebyshev shells of grid cells around the point's cell; after shell R
// every unvisited center is farther than (R - slack) * cell, so the search
// stops as soon as the best squared distance is below that bound (with a
// relative margin covering fp rounding of the cell indices and distances).
// When the next shell would hold more cells than there are centers the warp
// scans all centers instead.  Either way the result equals np.argmin over all
// centers.
__global__ void k_assign_fallback(const int32_t* rows, int64_t row_off,
                                  const double* __restrict__ pos, GridParams gp,
                                  CellIndex table, const double4* __restrict__ spos,
                                  const FbEntry* __restrict__ fb_list, const int32_t* fb_count,
                                  int32_t* __restrict__ assign, int32_t* __restrict__ far_list,
                                  int32_t* __restrict__ far_count,
                                  unsigned long long* __restrict__ far_d,
                                  int32_t* __restrict__ far_j) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int total = *fb_count;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < total; w += warps) {
    const FbEntry e = fb_list[w];
    const int64_t i = e.i;
    const int64_t r = class_row(rows, row_off, i);
    const double px = pos[r * 3], py = pos[r * 3 + 1], pz = pos[r * 3 + 2];
    const long long cx = cell_coord(px, gp.lo[0], gp.cell);
    const long long cy = cell_coord(py, gp.lo[1], gp.cell);
    const long long cz = cell_coord(pz, gp.lo[2], gp.cell);
    // the 27 cells' best, as k_assign_cells found it
    Best b{e.d2, e.j};
    bool resolved = false;
    long long spent = 27;  // cells enumerated; beyond kShellBudget the tiled scan is cheaper
    for (int R = 1;; ++R) {
      const double lim = (double(R) - gp.slack) * gp.cell;
      if (b.j != 0x7FFFFFFF && b.d2 < lim * lim * (1.0 - 1e-9)) {
        resolved = true;
        break;
      }
      const long long side = 2LL * R + 3;
      const long long cube = side * side * side;
      if (spent + cube > kShellBudget || R > gp.max_dim + 1) break;
      spent += cube;
      const int Rn = R + 1;
      for (long long t = lane; t < cube; t += 32) {
        const int dx = int(t / (side * side)) - Rn;
        const int dy = int((t / side) % side) - Rn;
        const int dz = int(t % side) - Rn;
        if (max(abs(dx), max(abs(dy), abs(dz))) != Rn) continue;
        const long long nx = cx + dx, ny = cy + dy, nz = cz + dz;
        if (nx < 0 || ny < 0 || nz < 0 || nx >= gp.dims[0] || ny >= gp.dims[1] ||
            nz >= gp.dims[2])
          continue;  // no center lives outside the class bounding grid
        scan_cell(gp, table, spos, nx, ny, nz, px, py, pz, b);
      }
      warp_best(b);
    }
    if (lane == 0) {
      if (resolved) assign[i] = b.j;
      else {
        const int slot = atomicAdd(far_count, 1);
        far_list[slot] = int32_t(i);
        far_d[slot] = ~0ULL;
        far_j[slot] = 0x7FFFFFFF;
      }
    }
  }
}

// Exact global argmin for the few points far from every center: blocks take
// (256 points) x (a slice of the centers), the slice is staged through shared
// memory and shared by all the block's points.  The slices merge through two
// atomics that keep the result lexicographic in (d2, center): pass 0 takes the
// min of d2 (non-negative doubles order like their bit patterns), pass 1 the
// lowest center attaining it.
constexpr int kFarSlices = 32;
__global__ void __launch_bounds__(256)
k_far_tiles(const int32_t* rows, int64_t row_off, const double* __restrict__ pos,
            const double4* __restrict__ spos, int m, const int32_t* __restrict__ far_list,
            const int32_t* __restrict__ far_count, unsigned long long* __restrict__ far_d,
            int32_t* __restrict__ far_j, int pass) {
  __shared__ double4 tile[256];
  const int nf = *far_count;
  const int groups = (nf + 255) / 256;
  // few far points: cut the centers into more slices so every block works
  const int slices = groups > 0 ? max(kFarSlices, int(gridDim.x) / groups) : kFarSlices;
  const int64_t per = (int64_t(m) + slices - 1) / slices;
  for (int blk = blockIdx.x; blk < groups * slices; blk += gridDim.x) {
    const int grp = blk / slices, slice = blk % slices;
    const int pi = grp * 256 + threadIdx.x;
    const bool active = pi < nf;
    double px = 0, py = 0, pz = 0, target = 0;
    if (active) {
      const int64_t r = class_row(rows, row_off, far_list[pi]);
      px = pos[r * 3];
      py = pos[r * 3 + 1];
      pz = pos[r * 3 + 2];
      if (pass) target = __longlong_as_double((long long)far_d[pi]);
    }
    Best b{INFINITY, 0x7FFFFFFF};
    const int64_t c0 = slice * per;
    const int64_t c1 = (c0 + per < int64_t(m)) ? c0 + per : int64_t(m);
    for (int64_t base = c0; base < c1; base += 256) {
      __syncthreads();
      if (base + threadIdx.x < c1) tile[threadIdx.x] = spos[base + threadIdx.x];
      __syncthreads();
      const int cnt = (c1 - base < 256) ? int(c1 - base) : 256;
      if (active) {
        if (pass == 0) {
          for (int q = 0; q < cnt; ++q) {
            const double4 c = tile[q];
            b.d2 = fmin(b.d2, dist2_exact(px, py, pz, c.x, c.y, c.z));
          }
        } else {
          for (int q = 0; q < cnt; ++q) {
            const double4 c = tile[q];
            if (dist2_exact(px, py, pz, c.x, c.y, c.z) == target)
              b.j = min(b.j, int(__double_as_longlong(c.w)));
          }
        }
      }
    }
    if (active) {
      if (pass == 0) atomicMin(&far_d[pi], (unsigned long long)__double_as_longlong(b.d2));
      else if (b.j != 0x7FFFFFFF) atomicMin(&far_j[pi], b.j);
    }
  }
}

__global__ void k_far_store(const int32_t* __restrict__ far_list, const int32_t* __restrict__ far_count,
                            const int32_t* __restrict__ far_j, int32_t* __restrict__ assign) {
  const int nf = *far_count;
  for (int pi = blockIdx.x * blockDim.x + threadIdx.x; pi < nf; pi += gridDim.x * blockDim.x)
    assign[far_list[pi]] = far_j[pi];
}

__global__ void k_group_values(const int32_t* rows, int64_t row_off, int64_t n, int32_t* out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = int32_t(class_row(rows, row_off, i));
}

__global__ void k_histogram(const int32_t* __restrict__ assign, int64_t n, int32_t* counts) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(&counts[assign[i]], 1);
}

struct SquareOp {
  __host__ __device__ int64_t operator()(int32_t s) const { return int64_t(s) * s; }
};
struct MaxOp {
  __host__ __device__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};

struct Oversize {
  const int32_t* counts;
  int32_t limit;
  __device__ bool operator()(int32_t j) const { return counts[j] > limit; }
};

// (group, count, start, center record) of the oversize groups, for the host.
__global__ void k_oversize_info(const int32_t* __restrict__ over, const int32_t* __restrict__ n_over,
                                const int32_t* __restrict__ counts,
                                const int32_t* __restrict__ gstart,
                                const int32_t* __restrict__ crec, int64_t* __restrict__ out) {
  const int n = *n_over;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int j = over[k];
    out[k * 4] = j;
    out[k * 4 + 1] = counts[j];
    out[k * 4 + 2] = gstart[j];
    out[k * 4 + 3] = crec[j];
  }
}

// Staging layout of the oversize groups: dst = exclusive scan of their sizes.
__global__ void k_oversize_seg(const int64_t* __restrict__ info, const int32_t* __restrict__ n_over,
                               const int64_t* __restrict__ dst, int64_t row_off,
                               int64_t* __restrict__ seg, int32_t* __restrict__ scalars) {
  const int n = *n_over;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    seg[k * 3] = row_off + info[k * 4 + 2];
    seg[k * 3 + 1] = info[k * 4 + 1];
    seg[k * 3 + 2] = dst[k];
    if (k == n - 1) scalars[3] = int32_t(dst[k] + info[k * 4 + 1]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && n == 0) scalars[3] = 0;
}

struct OverCount {
  const int64_t* info;
  __host__ __device__ int64_t operator()(int32_t k) const { return info[k * 4 + 1]; }
};

// Gather the members of the oversize groups for the host split loop: record
// id, position (SoA), squared distance to the group's center (fp64, the
// reference's rounding, like the host dist2) and the slot of the center
// among the members (slot_of[k], min over matches; >= staged means absent).
__global__ void k_gather_oversize(const int32_t* __restrict__ grp_rec,
                                  const int64_t* __restrict__ seg, const int32_t* __restrict__ n_seg,
                                  const int64_t* __restrict__ info, const double* __restrict__ pos,
                                  int32_t* __restrict__ out_rec, double* __restrict__ ox,
                                  double* __restrict__ oy, double* __restrict__ oz,
                                  double* __restrict__ od0, int32_t* __restrict__ slot_of) {
  // seg[k*3+0] = source offset, seg[k*3+1] = count, seg[k*3+2] = destination offset
  const int nk = *n_seg;
  for (int k = blockIdx.x; k < nk; k += gridDim.x) {
    const int64_t src = seg[k * 3], cnt = seg[k * 3 + 1], dst = seg[k * 3 + 2];
    const int32_t crec = int32_t(info[k * 4 + 3]);
    const double cx = pos[int64_t(crec) * 3], cy = pos[int64_t(crec) * 3 + 1],
                 cz = pos[int64_t(crec) * 3 + 2];
    for (int64_t t = threadIdx.x; t < cnt; t += blockDim.x) {
      const int32_t r = grp_rec[src + t];
      const double px = pos[int64_t(r) * 3], py = pos[int64_t(r) * 3 + 1], pz = pos[int64_t(r) * 3 + 2];
      out_rec[dst + t] = r;
      ox[dst + t] = px;
      oy[dst + t] = py;
      oz[dst + t] = pz;
      od0[dst + t] = dist2_exact(px, py, pz, cx, cy, cz);
      if (r == crec) atomicMin(&slot_of[k], int32_t(dst + t));
    }
  }
}

// First-split outcomes of every oversize group for every possible pick: bit
// m of row p of group k = (member m is strictly closer to member p than to
// the group's center), i.e. "m moves if p is the new center"
// (clustering.py:69-74) with the host loop's exact fp64 distances.  82% of
// the split loop's splits are first splits; with these rows the host only
// draws the pick and partitions.  mask_off = exclusive scan of
// cnt * ceil(cnt / 64) words (MaskWords).
struct MaskWords {
  const int64_t* info;
  const int32_t* n_over;
  __host__ __device__ int64_t operator()(int32_t k) const {
    if (k >= *n_over) return 0;
    const int64_t cnt = info[k * 4 + 1];
    return cnt * ((cnt + 63) / 64);
  }
};

// Mask total, and the bulk staging's transfer pieces: piece j holds the
// oversize groups [n*j/P, n*(j+1)/P) -- bounds[j] = {first group, its staged
// offset, its mask offset}, bounds[P] the totals.
constexpr int kBulkPieces = 8;
__global__ void k_mask_total(const int64_t* __restrict__ mask_off, const int64_t* __restrict__ info,
                             const int32_t* __restrict__ n_over, const int64_t* __restrict__ seg,
                             int64_t* __restrict__ total) {
  const int n = *n_over;
  int64_t* bounds = total + 1;
  if (n == 0) {
    *total = 0;
    for (int j = 0; j <= kBulkPieces; ++j) bounds[3 * j] = bounds[3 * j + 1] = bounds[3 * j + 2] = 0;
    return;
  }
  const int64_t cnt = info[(n - 1) * 4 + 1];
  *total = mask_off[n - 1] + cnt * ((cnt + 63) / 64);
  for (int j = 0; j <= kBulkPieces; ++j) {
    const int64_t gk = int64_t(n) * j / kBulkPieces;
    bounds[3 * j] = gk;
    bounds[3 * j + 1] = gk < n ? seg[gk * 3 + 2] : seg[(n - 1) * 3 + 2] + cnt;
    bounds[3 * j + 2] = gk < n ? mask_off[gk] : *total;
  }
}

__global__ void k_first_split_masks(const int64_t* __restrict__ seg, const int32_t* __restrict__ n_over,
                                    const int64_t* __restrict__ mask_off,
                                    const double* __restrict__ x, const double* __restrict__ y,
                                    const double* __restrict__ z, const double* __restrict__ d0,
                                    unsigned long long* __restrict__ masks,
                                    int32_t* __restrict__ moved) {
  const int nk = *n_over;
  for (int k = blockIdx.x; k < nk; k += gridDim.x) {
    const int64_t cnt = seg[k * 3 + 1], b = seg[k * 3 + 2];
    const int64_t words = (cnt + 63) / 64;
    unsigned long long* mk = masks + mask_off[k];
    for (int64_t item = threadIdx.x; item < cnt * words; item += blockDim.x) {
      const int64_t p = item / words, w = item - p * words;
      const double px = x[b + p], py = y[b + p], pz = z[b + p];
      unsigned long long bits = 0;
      const int64_t m0 = w * 64, m1 = m0 + 64 < cnt ? m0 + 64 : cnt;
      for (int64_t mm = m0; mm < m1; ++mm)
        if (dist2_exact(x[b + mm], y[b + mm], z[b + mm], px, py, pz) < d0[b + mm])
          bits |= 1ull << (mm - m0);
      mk[item] = bits;
      // the size of the moved half for pick p (moved[] zeroed beforehand)
      if (bits) atomicAdd(&moved[b + p], __popcll(bits));
    }
  }
}

// The first splits the host booked without moving members (DeferredSplit:
// staged begin, size, pick's mask row): stable partition of the staged
// record ids in place, kept members first, then the moved ones -- exactly
// the host's partition.  Block per split, <= 3 members per thread.
constexpr int kApplyThreads = 128;
__global__ void __launch_bounds__(kApplyThreads)
k_apply_first_splits(const int64_t* __restrict__ dsplit, int64_t n_split,
                     const unsigned long long* __restrict__ masks, int32_t* __restrict__ ids) {
  for (int64_t i = blockIdx.x; i < n_split; i += gridDim.x) {
    const int64_t b = dsplit[3 * i], sz = dsplit[3 * i + 1];
    const unsigned long long* row = masks + dsplit[3 * i + 2];
    const int words = int((sz + 63) / 64);
    int moved_total = 0;
    for (int w = 0; w < words; ++w) moved_total += __popcll(row[w]);
    const int kept_total = int(sz) - moved_total;
    int32_t v[3];
    int dst[3];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int t = threadIdx.x + u * kApplyThreads;
      dst[u] = -1;
      if (t < sz) {
        v[u] = ids[b + t];
        const int w = t >> 6;
        int before = __popcll(row[w] & ((1ull << (t & 63)) - 1ull));
        for (int w2 = 0; w2 < w; ++w2) before += __popcll(row[w2]);
        const bool f = (row[w] >> (t & 63)) & 1ull;
        dst[u] = f ? kept_total + before : t - before;
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 3; ++u)
      if (dst[u] >= 0) ids[b + dst[u]] = v[u];
    __syncthreads();
  }
}

// ------------------------------------------------------------ layout
// Internal cluster order: part A = every group that needed no split, class by
// class in group order; part B = the split loop's results (modified groups and
// split-off groups).  Part A is laid out, packed and aggregated on the device
// while the host runs the split loop; the reference's numbering (groups in
// order, skipping empty ones, split-off groups appended per class,
// clustering.py:87-93) is kept in ref_of.
struct LayoutAcc {  // exclusive-scan element over a class's groups
  int32_t a, ne, rows;
  int64_t w;
};
struct LayoutSum {
  __host__ __device__ LayoutAcc operator()(const LayoutAcc& x, const LayoutAcc& y) const {
    return LayoutAcc{x.a + y.a, x.ne + y.ne, x.rows + y.rows, x.w + y.w};
  }
};
struct LayoutOf {
  int32_t max_size;
  __host__ __device__ LayoutAcc operator()(int32_t size) const {
    const bool in_a = size > 0 && size <= max_size;
    return LayoutAcc{in_a ? 1 : 0, size > 0 ? 1 : 0, in_a ? size : 0,
                     in_a ? ((int64_t(size) * size + 3) & ~int64_t(3)) : 0};
  }
};

struct LayoutOfPerm {  // LayoutOf of the groups taken in layout order
  const int32_t* counts;
  const int32_t* order;
  int32_t max_size;
  __host__ __device__ LayoutAcc operator()(int32_t i) const {
    return LayoutOf{max_size}(counts[order[i]]);
  }
};

// Device totals: acc = {A clusters, A rows, A kernel floats, non-empty groups}.
// cls = per class {A begin, A end, reference base, non-empty groups}.
__global__ void k_layout_a(const int32_t* __restrict__ counts, const int32_t* __restrict__ gstart,
                           const int32_t* __restrict__ crec, const LayoutAcc* __restrict__ pre,
                           const int32_t* __restrict__ order, const LayoutAcc* __restrict__ pre_o,
                           int m, int32_t max_size, int64_t row_off, int64_t appended_before,
                           const int64_t* __restrict__ acc, int32_t* __restrict__ cl_off,
                           int32_t* __restrict__ cl_size, int64_t* __restrict__ w_off,
                           int64_t* __restrict__ cl_src, int32_t* __restrict__ cl_center,
                           int32_t* __restrict__ ref_of, int32_t* __restrict__ ne_prefix) {
  // i walks the layout order; pre_o is the layout scan, pre (group order) the
  // reference numbering's count of non-empty groups before j
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int j = order[i];
    const int32_t size = counts[j];
    const int32_t ne = pre[j].ne;
    ne_prefix[j] = ne;
    if (size <= 0 || size > max_size) continue;
    const LayoutAcc e = pre_o[i];
    const int64_t k = acc[0] + e.a;
    cl_off[k] = int32_t(acc[1] + e.rows);
    cl_size[k] = size;
    w_off[k] = acc[2] + e.w;
    cl_src[k] = row_off + gstart[j];
    cl_center[k] = crec[j];
    ref_of[k] = int32_t(acc[3] + appended_before + ne);
  }
}

__global__ void k_layout_a_totals(const int32_t* __restrict__ counts,
                                  const LayoutAcc* __restrict__ pre, int m, int32_t max_size,
                                  int64_t appended_before, int64_t* __restrict__ acc,
                                  int64_t* __restrict__ cls) {
  const LayoutAcc last = LayoutSum()(pre[m - 1], LayoutOf{max_size}(counts[m - 1]));
  cls[0] = acc[0];
  cls[1] = acc[0] + last.a;
  cls[2] = acc[3] + appended_before;
  cls[3] = last.ne;
  acc[0] += last.a;
  acc[1] += last.rows;
  acc[2] += last.w;
  acc[3] += last.ne;
}

// Part B: b[t*8..] = {class, group j (>= 0) or -(1+appended index), size, row
// offset in part B, kernel offset in part B, split-buffer offset, center, 0}.
__global__ void k_layout_b(const int64_t* __restrict__ b, int64_t nb, const int64_t* __restrict__ acc,
                           const int64_t* __restrict__ cls, const int32_t* __restrict__ ne_prefix_all,
                           const int64_t* __restrict__ class_center_off, int32_t* __restrict__ cl_off,
                           int32_t* __restrict__ cl_size, int64_t* __restrict__ w_off,
                           int64_t* __restrict__ cl_src, int32_t* __restrict__ cl_center,
                           int32_t* __restrict__ ref_of) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < nb;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t* e = b + t * 8;
    const int c = int(e[0]);
    const int64_t k = acc[0] + t;
    cl_off[k] = int32_t(acc[1] + e[3]);
    cl_size[k] = int32_t(e[2]);
    w_off[k] = acc[2] + e[4];
    cl_src[k] = -1 - e[5];
    cl_center[k] = int32_t(e[6]);
    const int64_t* ci = cls + 4 * c;
    ref_of[k] = int32_t(e[1] >= 0 ? ci[2] + ne_prefix_all[class_center_off[c] + e[1]]
                                  : ci[2] + ci[3] + (-1 - e[1]));
  }
}

// Closing offsets cl_off[M], w_off[M] and the internal range of part B.
__global__ void k_layout_close(int64_t nb, int64_t rows_b, int64_t w_b, const int64_t* __restrict__ acc,
                               int32_t* __restrict__ cl_off, int64_t* __restrict__ w_off,
                               int64_t* __restrict__ range_b) {
  const int64_t M = acc[0] + nb;
  cl_off[M] = int32_t(acc[1] + rows_b);
  w_off[M] = acc[2] + w_b;
  range_b[0] = acc[0];
  range_b[1] = M;
}

// Cluster-major permutation for the clusters in [range[0], range[1]): warp
// per cluster copies its member list; records get their position and the
// reference cluster number.
__global__ void k_fill_perm(const int64_t* __restrict__ range, const int32_t* __restrict__ cl_off,
                            const int32_t* __restrict__ cl_size, const int64_t* __restrict__ cl_src,
                            const int32_t* __restrict__ ref_of, const int32_t* __restrict__ grp_rec,
                            const int32_t* __restrict__ split_rec, int32_t* __restrict__ perm,
                            int32_t* __restrict__ clpos, int32_t* __restrict__ cluster_id) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t k1 = range[1];
  for (int64_t k = range[0] + ((blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5); k < k1;
       k += warps) {
    const int32_t q0 = cl_off[k], sz = cl_size[k];
    const int64_t src = cl_src[k];
    const int32_t* from = src >= 0 ? grp_rec + src : split_rec + (-1 - src);
    const int32_t ref = ref_of[k];
    for (int32_t t = lane; t < sz; t += 32) {
      const int32_t r = from[t];
      perm[q0 + t] = r;
      clpos[r] = q0 + t;
      if (cluster_id) cluster_id[r] = ref;
    }
  }
}

__global__ void k_invert_ref(const int32_t* __restrict__ ref_of, int64_t m,
                             int32_t* __restrict__ internal_of) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < m;
       k += int64_t(gridDim.x) * blockDim.x)
    internal_of[ref_of[k]] = int32_t(k);
}

template <class T>
void to_host(std::vector<T>& h, const T* d, size_t n, cudaStream_t s) {
  h.resize(n);
  if (n) VPG_CUDA(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  count_transfer(0, n * sizeof(T));
}
template <class T>
void to_device(T* d, const std::vector<T>& h, cudaStream_t s) {
  if (!h.empty())
    VPG_CUDA(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  count_transfer(h.size() * sizeof(T), 0);
}

// Host -> device copies that must not queue behind a bulk transfer on the
// copy engine (the async record upload the build overlaps): the kernel reads
// the pinned host buffer directly (UVA-mapped) instead of a memcpy.
// Kernel copy out of pinned host memory (PCIe reads, no copy-engine queue):
// 16-byte reads when both sides allow it, so fewer requests are in flight.
__global__ void k_copy_host(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                            int64_t words) {
  const int64_t tid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t head = 0;
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    const int64_t quads = words / 4;
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (int64_t i = tid; i < quads; i += stride) d4[i] = s4[i];
    head = quads * 4;
  }
  for (int64_t i = head + tid; i < words; i += stride) dst[i] = src[i];
}

// Copy of a pinned host array that a host thread is still writing: chunk c
// (kReadyChunk words) is read once ready[c] (host memory) is set; the host
// thread sets it after the chunk's words (release).  The words are read with
// ld.relaxed.sys (never the non-coherent path: the host writes them while the
// kernel runs), and the wait is bounded: a host thread that has not
// published a chunk within kReadyTimeoutNs aborts the launch (an error on the
// stream, never a hung GPU).
constexpr int64_t kReadyChunk = 8192;
constexpr unsigned long long kReadyTimeoutNs = 30ull * 1000 * 1000 * 1000;
__global__ void k_copy_when_ready(const uint32_t* src, const int32_t* ready,
                                  uint32_t* __restrict__ dst, int64_t words) {
  const int64_t chunks = (words + kReadyChunk - 1) / kReadyChunk;
  for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    if (threadIdx.x == 0) {
      int v = 0;
      unsigned long long t0, t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      do {
        asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(ready + c) : "memory");
        if (!v) {
          __nanosleep(500);
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
          if (t - t0 > kReadyTimeoutNs) __trap();
        }
      } while (!v);
    }
    __syncthreads();
    const int64_t b = c * kReadyChunk, e = min(words, b + kReadyChunk);
    // 16-byte relaxed loads (chunk starts are 16-byte aligned), a word tail
    const int64_t e4 = b + ((e - b) & ~int64_t(3));
    for (int64_t i = b + 4 * int64_t(threadIdx.x); i < e4; i += 4 * int64_t(blockDim.x)) {
      uint4 w;
      asm volatile("ld.relaxed.sys.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w) : "l"(src + i) : "memory");
      *reinterpret_cast<uint4*>(dst + i) = w;
    }
    for (int64_t i = e4 + threadIdx.x; i < e; i += blockDim.x) {
      uint32_t w;
      asm volatile("ld.relaxed.sys.global.b32 %0, [%1];" : "=r"(w) : "l"(src + i) : "memory");
      dst[i] = w;
    }
    __syncthreads();
  }
}

struct HostUpload {
  std::vector<std::unique_ptr<HostBuf<uint32_t>>> keep;  // alive until the build syncs
  // source already pinned (HostBuf): no staging copy
  template <class T>
  void pinned(T* d, const T* h, size_t n, cudaStream_t s) {
    static_assert(sizeof(T) % 4 == 0, "word-sized elements");
    const int64_t words = int64_t(n * sizeof(T) / 4);
    if (!words) return;
    VPG_LAUNCH(k_copy_host, grid_for(words, 256, 1024), 256, 0, s,
               reinterpret_cast<const uint32_t*>(h), reinterpret_cast<uint32_t*>(d), words);
    count_transfer(n * sizeof(T), 0);
  }
  template <class T>
  void put(T* d, const T* h, size_t n, cudaStream_t s) {
    if (!n) return;
    keep.emplace_back(new HostBuf<uint32_t>((n * sizeof(T) + 3) / 4));
    std::memcpy(keep.back()->get(), h, n * sizeof(T));
    pinned(d, reinterpret_cast<const T*>(keep.back()->get()), n, s);
  }
};

int bits_for(uint64_t max_value) {
  int b = 1;
  while (b < 64 && (max_value >> b)) ++b;
  return b;
}

// cells of the dense packed key space, and whether a direct cell index over it
// is small enough (8 bytes per cell)
int64_t dense_cells(const GridParams& gp) {
  return int64_t(gp.dims[0] + 4) * int64_t(gp.dims[1] + 4) * int64_t(gp.dims[2] + 4);
}
bool dense_cells_ok(const GridParams& gp, int64_t m) {
  if (!gp.packed) return false;
  const double cells = double(gp.dims[0] + 4) * double(gp.dims[1] + 4) * double(gp.dims[2] + 4);
  return cells <= 8.0 * double(m) + 65536.0;
}

// radix bits of the dense packed cell keys (cell_key)
int packed_key_bits(const GridParams& gp) {
  const double cells = double(gp.dims[0] + 4) * double(gp.dims[1] + 4) * double(gp.dims[2] + 4);
  return cells < 1.8e19 ? bits_for(uint64_t(cells)) : 64;
}

struct StageClock {
  bool on;
  cudaStream_t s;
  std::chrono::steady_clock::time_point t0;
  double* slots;
  StageClock(bool enabled, cudaStream_t st, double* out) : on(enabled), s(st), slots(out) {
    if (on) {
      cudaStreamSynchronize(s);
      t0 = std::chrono::steady_clock::now();
    }
  }
  void mark(int slot) {
    if (!on) return;
    cudaStreamSynchronize(s);
    auto t1 = std::chrono::steady_clock::now();
    slots[slot] += std::chrono::duration<double, std::milli>(t1 - t0).count();
    t0 = t1;
  }
};

// A non-blocking stream per device for host transfers that must not hold up
// the compute stream.
cudaStream_t side_stream(int which = 0) {
  static cudaStream_t streams[2][64] = {};
  int dev = 0;
  VPG_CUDA(cudaGetDevice(&dev));
  cudaStream_t& st = streams[which][dev];
  if (!st) {
    // the highest priority: the oversize staging and part B feed the host
    // split loop and the critical path, their blocks go first whenever an
    // SM frees up
    int lo = 0, hi = 0;
    VPG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    VPG_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, hi));
  }
  return st;
}

template <class F>
void cub_call(F&& f, cudaStream_t s) {
  size_t bytes = 0;
  VPG_CUDA(f(nullptr, bytes));
  void* tmp = scratch(s, "cub_temp", bytes + 256);
  const int tok = profiling() ? prof_begin("cub", s) : -1;
  VPG_CUDA(f(tmp, bytes));
  if (tok >= 0) prof_end(tok, s);
  count_launch(2);
}

// The points bucketed by cell for k_assign_cells: ids in cell order (the
// octant in the top bits when oct_in_ids), one run per occupied cell, the run
// count in *n_runs (device).  A counting sort over the dense packed cell keys
// when the padded grid is small; a radix sort of the (hashed) keys otherwise.
struct PointCells {
  int32_t *pids_sorted, *run_start, *run_len;
  bool oct_in_ids;
};
PointCells sort_points_by_cell(const int32_t* rows_p, int64_t row_off, int64_t n, const double* pos,
                               const GridParams& gp, int32_t* n_runs, const std::string& tag,
                               cudaStream_t s) {
  const int block = 256;
  PointCells pc{};
  auto* pkeys = scratch_of<unsigned long long>(s, (tag + "pkeys").c_str(), n);
  auto* pkeys_sorted = scratch_of<unsigned long long>(s, (tag + "pkeys_sorted").c_str(), n);
  int32_t* pids = scratch_of<int32_t>(s, (tag + "pids").c_str(), n);
  pc.pids_sorted = scratch_of<int32_t>(s, (tag + "pids_sorted").c_str(), n);
  pc.run_start = scratch_of<int32_t>(s, (tag + "run_start").c_str(), n + 1);
  pc.run_len = scratch_of<int32_t>(s, (tag + "run_len").c_str(), n + 1);
  const double cells = double(gp.dims[0] + 4) * double(gp.dims[1] + 4) * double(gp.dims[2] + 4);
  if (gp.packed && cells <= 4.0 * double(n) + 4096.0 && cells < 2.0e9) {
    const int64_t nc = int64_t(cells);
    int32_t* counts = scratch_of<int32_t>(s, (tag + "cell_counts").c_str(), size_t(nc) + 1);
    int32_t* offs = scratch_of<int32_t>(s, (tag + "cell_offs").c_str(), size_t(nc) + 1);
    int32_t* pkey = reinterpret_cast<int32_t*>(pkeys);
    uint8_t* poct = nullptr;  // octants (fewer than 2^29 points only)
    if (n < (int64_t(1) << kOctShift)) poct = scratch_of<uint8_t>(s, (tag + "cell_oct").c_str(), n);
    pc.oct_in_ids = poct != nullptr;
    VPG_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * (nc + 1), s));
    VPG_LAUNCH(k_cell_count, grid_for(n, block, 1 << 30), block, 0, s, rows_p, row_off, n, pos, gp, counts,
               pkey, poct);
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(t, b, counts, offs, int(nc + 1), s);
    }, s);
    VPG_LAUNCH(k_cell_scatter, grid_for(n, block, 1 << 30), block, 0, s, n, pkey, poct, offs, counts,
               pc.pids_sorted);
    int32_t* sel = reinterpret_cast<int32_t*>(pkeys_sorted);
    cub::CountingInputIterator<int32_t> ci(0);
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceSelect::If(t, b, ci, sel, n_runs, int(nc), CellNonEmpty{offs}, s);
    }, s);
    VPG_LAUNCH(k_cell_runs, grid_for(n, block), block, 0, s, sel, n_runs, offs, pc.run_start,
               pc.run_len);
  } else {
    const int end_bits = gp.packed ? packed_key_bits(gp) : 64;
    VPG_LAUNCH(k_point_keys, grid_for(n, block), block, 0, s, rows_p, row_off, n, pos, gp, pkeys,
               pids);
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, pkeys, pkeys_sorted, pids, pc.pids_sorted,
                                             int(n), 0, end_bits, s);
    }, s);
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRunLengthEncode::Encode(t, b, pkeys_sorted, pkeys, pc.run_len, n_runs,
                                                int(n), s);
    }, s);
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(t, b, pc.run_len, pc.run_start, int(n), s);
    }, s);
  }
  return pc;
}

// VPG_DEBUG_TIMING=1 prints sub-stage wall times of the build to stderr.
struct DebugClock {
  bool on;
  cudaStream_t s;
  std::chrono::steady_clock::time_point t0;
  explicit DebugClock(cudaStream_t st) : on(getenv("VPG_DEBUG_TIMING") != nullptr), s(st) {
    t0 = std::chrono::steady_clock::now();
  }
  void mark(const char* what, bool sync = true) {
    if (!on) return;
    if (sync) cudaStreamSynchronize(s);
    const auto t1 = std::chrono::steady_clock::now();
    fprintf(stderr, "[vpg] %-28s %8.3f ms\n", what,
            std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};

struct ClassPlan {
  int64_t n, row_off, m, center_off;
  double lo[3], hi[3];
};

// The reference's grid for one class: lo/cell as clustering.py:102-106 (host
// fp64, glibc pow like Python's float pow), plus the device table geometry.
GridParams make_grid(const ClassPlan& p) {
  GridParams gp{};
  gp.m = int(p.m);
  double extent[3];
  for (int a = 0; a < 3; ++a) {
    extent[a] = p.hi[a] - p.lo[a];
    gp.lo[a] = p.lo[a];
  }
  double volume = std::max(extent[0], 1e-12) * std::max(extent[1], 1e-12);
  volume = volume * std::max(extent[2], 1e-12);
  gp.cell = std::max(std::pow(volume / double(p.m), 1.0 / 3.0), 1e-9);
  bool fits = true;
  gp.max_dim = 0;
  for (int a = 0; a < 3; ++a) {
    const double d = std::floor(extent[a] / gp.cell) + 2.0;
    fits = fits && (d + 2.0 < 2097152.0);
    gp.dims[a] = d < 9.0e18 ? (long long)d : (long long)9.0e18;
    gp.max_dim = std::max(gp.max_dim, gp.dims[a]);
  }
  gp.packed = fits ? 1 : 0;
  // u = (p-lo)/cell carries a relative error of a few ulp; allow 2^-44 * |u|
  gp.slack = 2.0 * (double(std::min<long long>(gp.max_dim, 1LL << 52)) + 4.0) * 5.7e-14;
  uint64_t cap = 1024;
  while (cap < uint64_t(p.m) * 2) cap <<= 1;
  gp.table_mask = cap - 1;
  return gp;
}

}  // namespace

void build_graph(vpg_graph* g, const vpg_records& rec, int32_t K, vpg_pcg64* rng_state,
                 bool timings, bool with_ops, cudaStream_t s, cudaEvent_t fields_ready) {
  const int64_t n = rec.n;
  VPG_REQUIRE(K >= 1, VPG_EINVAL, "cluster size K must be >= 1");
  VPG_REQUIRE(n < (int64_t(1) << 31) - 1, VPG_ELIMIT, "more than 2^31-2 records per device");
  g->n = n;
  g->K = K;
  for (double& t : g->info.build_ms) t = 0.0;
  StageClock clk(timings, s, g->info.build_ms);
  HostUpload up;
  std::vector<std::unique_ptr<HostBuf<int32_t>>> up_hold;  // pinned inputs of queued kernels
  Pcg64 rng(*rng_state);
  const int block = 256;

  g->perm.alloc(n, s);
  g->clpos.alloc(n, s);
  g->cluster_id.alloc(n, s);
  g->cluster_id_ready = false;  // filled on first export (ensure_cluster_ids)
  if (n == 0) {
    g->m = 0;
    for (auto* v : {&g->cl_off, &g->cl_size, &g->cl_center, &g->ref_of, &g->internal_of}) {
      v->alloc(1, s);
      VPG_CUDA(cudaMemsetAsync(v->get(), 0, sizeof(int32_t), s));
    }
    g->w_off.alloc(1, s);
    VPG_CUDA(cudaMemsetAsync(g->w_off.get(), 0, sizeof(int64_t), s));
    if (with_ops) alloc_operator_buffers(g, 1, s);
    g->chunk_first.alloc(1, s);
    VPG_CUDA(cudaMemsetAsync(g->chunk_first.get(), 0, sizeof(int32_t), s));
    g->n_chunks_dev.alloc(1, s);
    VPG_CUDA(cudaMemsetAsync(g->n_chunks_dev.get(), 0, sizeof(int64_t), s));
    rng.store(rng_state);
    return;
  }
  VPG_CUDA(cudaMemsetAsync(g->clpos.get(), 0xFF, sizeof(int32_t) * n, s));  // -1: not placed

  // The center draw of a single-class record set (the common case) does not
  // need the class pass: a host thread draws its swap targets speculatively
  // while the device finds the classes, and the draw is kept when there
  // turns out to be one class (else discarded, the generator untouched).
  struct SpecDraw {
    std::thread th;
    std::unique_ptr<HostBuf<int32_t>> targets, ready;  // ready[c]: chunk c written
    Pcg64 g;
    int64_t steps = 0;
    bool adopted = false;  // the build uses it: rng takes g once the thread ends
    explicit SpecDraw(const Pcg64& r) : g(r) {}
    ~SpecDraw() {
      if (th.joinable()) th.join();
    }
  } spec(rng);
  // before the host draws again: a speculative draw in use hands over its state
  auto rng_ready = [&]() {
    if (spec.th.joinable()) spec.th.join();
    if (spec.adopted) {
      rng = spec.g;
      spec.adopted = false;
    }
  };
  {
    const int64_t m_all = (n + K - 1) / K;
    if (n > 10000 && m_all > n / 50) {
      spec.steps = n - std::max<int64_t>(n - m_all, 1);
      spec.targets.reset(new HostBuf<int32_t>(size_t(spec.steps) + 1));
      const int64_t chunks = (spec.steps + kReadyChunk - 1) / kReadyChunk;
      spec.ready.reset(new HostBuf<int32_t>(size_t(chunks) + 1));
      std::memset(spec.ready->get(), 0, sizeof(int32_t) * size_t(chunks + 1));
      spec.th = std::thread([&spec, n, chunks] {
        int32_t* t = spec.targets->get();
        volatile int32_t* rd = spec.ready->get();
        for (int64_t c = 0; c < chunks; ++c) {
          const int64_t e = std::min(spec.steps, (c + 1) * kReadyChunk);
          for (int64_t k = c * kReadyChunk; k < e; ++k)
            t[k] = int32_t(spec.g.bounded(uint64_t(n - 1 - k)));
          std::atomic_thread_fence(std::memory_order_release);
          rd[c] = 1;
        }
      });
    }
  }

  // ---- classes (np.unique order of kind<<32 | class_id, graph.py:59)
  const int nbits_words = 2 * kSlotsPerKind / 32;
  DBuf<uint32_t> bitmap(nbits_words + 1, s);
  VPG_CUDA(cudaMemsetAsync(bitmap.get(), 0, bitmap.bytes(), s));
  int32_t* d_err = reinterpret_cast<int32_t*>(bitmap.get() + nbits_words);
  VPG_LAUNCH(k_class_bitmap, grid_for(n, block), block, 0, s, rec.kind, rec.class_id, n,
             bitmap.get(), d_err);
  std::vector<uint32_t> h_bitmap;
  to_host(h_bitmap, bitmap.get(), nbits_words + 1, s);
  VPG_CUDA(cudaStreamSynchronize(s));
  VPG_REQUIRE(h_bitmap[nbits_words] == 0, VPG_ELIMIT,
              "record kind must be 0/1 and class_id in [0, 65536)");
  std::vector<uint32_t> slots;
  for (uint32_t w = 0; w < uint32_t(nbits_words); ++w)
    for (uint32_t b = 0; b < 32; ++b)
      if (h_bitmap[w] >> b & 1u) slots.push_back(w * 32 + b);
  const int n_cls = int(slots.size());
  VPG_REQUIRE(n_cls <= kMaxClasses, VPG_ELIMIT, "more than 256 compatibility classes");
  g->info.n_classes = n_cls;

  DBuf<uint32_t> d_slots(n_cls, s);
  up.put(d_slots.get(), slots.data(), slots.size(), s);
  DBuf<unsigned long long> stats(n_cls * 7, s);
  {
    std::vector<unsigned long long> init(n_cls * 7);
    for (int c = 0; c < n_cls; ++c) {
      init[c] = 0;
      for (int a = 0; a < 3; ++a) {
        init[n_cls + c * 3 + a] = ~0ull;
        init[4 * n_cls + c * 3 + a] = 0ull;
      }
    }
    up.put(stats.get(), init.data(), init.size(), s);
  }
  DBuf<uint8_t> cls_idx;
  if (n_cls > 1) cls_idx.alloc(n, s);
  VPG_LAUNCH(k_class_stats, grid_for(n, block, sm_count() * 4), block, 0, s, rec.kind,
             rec.class_id, rec.pos, n, d_slots.get(), n_cls, cls_idx.get(), stats.get(),
             stats.get() + n_cls, stats.get() + 4 * n_cls);
  // whether any cluster can store a W block (only when the record fields
  // are already resident: with an upload in flight, g is not there yet and
  // the full reservation stays)
  DBuf<int32_t> needs_w_dev;
  int32_t needs_w = 1;
  if (with_ops && !fields_ready) {
    needs_w_dev.alloc(1, s);
    launch_needs_stored_w(rec, needs_w_dev.get(), s);
    // (to pageable memory: returns once the copy has completed)
    VPG_CUDA(cudaMemcpyAsync(&needs_w, needs_w_dev.get(), sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    count_transfer(0, sizeof(int32_t));
  }
  std::vector<unsigned long long> h_stats;
  to_host(h_stats, stats.get(), n_cls * 7, s);

  // stable partition of record ids by class (np.nonzero(class_keys == key))
  DBuf<int32_t> rows;
  if (n_cls > 1) {
    DBuf<int32_t> iota(n, s);
    DBuf<uint8_t> cls_sorted(n, s);
    rows.alloc(n, s);
    VPG_LAUNCH(k_iota, grid_for(n, block), block, 0, s, iota.get(), n);
    const int end_bit = bits_for(uint64_t(n_cls - 1));
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, cls_idx.get(), cls_sorted.get(), iota.get(),
                                             rows.get(), int(n), 0, end_bit, s);
    }, s);
  }
  VPG_CUDA(cudaStreamSynchronize(s));
  clk.mark(0);

  std::vector<ClassPlan> plan(n_cls);
  int64_t row_off = 0, center_total = 0;
  for (int c = 0; c < n_cls; ++c) {
    ClassPlan& p = plan[c];
    p.n = int64_t(h_stats[c]);
    p.row_off = row_off;
    row_off += p.n;
    p.m = (p.n + K - 1) / K;
    p.center_off = center_total;
    center_total += p.m;
    for (int a = 0; a < 3; ++a) {
      p.lo[a] = order_key_inv(h_stats[n_cls + c * 3 + a]);
      p.hi[a] = order_key_inv(h_stats[4 * n_cls + c * 3 + a]);
    }
  }

  // per-class working storage (records grouped by center, class by class)
  int32_t* grp_rec = scratch_of<int32_t>(s, "grp_rec", n);
  int32_t* assign_all = scratch_of<int32_t>(s, "assign", n);
  int32_t* values = scratch_of<int32_t>(s, "values", n);
  FbEntry* fb_list = scratch_of<FbEntry>(s, "fb_list", n);
  DBuf<int32_t> counts_all(center_total, s), crec_all(center_total, s), gstart_all(center_total, s);
  DBuf<int32_t> ne_prefix_all(center_total + 1, s);
  DBuf<int32_t> scalars(4, s);  // fb count, n_runs, n_over
  DBuf<int32_t> far_count(1, s);
  DBuf<int64_t> mask_total(1 + 3 * (kBulkPieces + 1), s);
  DBuf<int64_t> acc(8, s), cls_info(size_t(4) * n_cls + 4, s), ranges(size_t(2) * n_cls + 2, s);
  DBuf<int64_t> class_center_off(n_cls + 1, s);
  VPG_CUDA(cudaMemsetAsync(counts_all.get(), 0, counts_all.bytes(), s));
  VPG_CUDA(cudaMemsetAsync(acc.get(), 0, acc.bytes(), s));
  {
    std::vector<int64_t> cco(n_cls + 1, 0);
    for (int c = 0; c < n_cls; ++c) cco[c] = plan[c].center_off;
    up.put(class_center_off.get(), cco.data(), cco.size(), s);
  }
  const int64_t max_size = 2 * int64_t(K);
  const int S = int(std::max<int64_t>(1, std::min<int64_t>(max_size, n)));

  // part A cluster arrays (at most one cluster per center)
  const int64_t cap_a = center_total + 1;
  DBuf<int32_t> a_off(cap_a, s), a_size(cap_a, s), a_center(cap_a, s), a_ref(cap_a, s);
  DBuf<int64_t> a_w(cap_a, s), a_src(cap_a, s);
  // the operator passes run against g's arrays: point them at part A for now
  g->cl_off = std::move(a_off);
  g->cl_size = std::move(a_size);
  g->cl_center = std::move(a_center);
  g->ref_of = std::move(a_ref);
  g->w_off = std::move(a_w);
  void* members = nullptr;
  if (with_ops) {
    // kernel blocks: sum of pad4(s^2) <= 2K * N + 3 per cluster, when any
    // cluster stores one
    const int64_t wt_cap =
        needs_w ? std::min<int64_t>(max_size, n) * n + 4 * (center_total + n) + 16 : 16;
    alloc_operator_buffers(g, wt_cap, s);
    members = scratch(s, "members", member_bytes() * size_t(n) + 256);
  }

  // per class: the split groups' members back to back, and 8 int64 per split
  // group (see k_layout_b) -- kept in the pinned buffers they were produced
  // in, so part B reads them from the device without host-side concatenation
  struct SplitChunk {
    std::unique_ptr<HostBuf<int32_t>> rec;
    int64_t n_rec;
    std::unique_ptr<HostBuf<int64_t>> b;
    int64_t n_b;
    std::unique_ptr<HostBuf<int64_t>> deferred;  // DeferredSplit triples
    int64_t n_deferred;
    std::unique_ptr<DBuf<unsigned long long>> masks;  // the class's first-split rows
  };
  std::vector<SplitChunk> chunks;
  int64_t split_total = 0, nb_total = 0;
  int64_t rows_b = 0, w_b = 0, appended_before = 0;
  int64_t n_splits = 0;
  HostBuf<int64_t> h_acc(8);
  cudaEvent_t acc_ready;
  VPG_CUDA(cudaEventCreateWithFlags(&acc_ready, cudaEventDisableTiming));
  cudaEvent_t placed, b_done;
  VPG_CUDA(cudaEventCreateWithFlags(&placed, cudaEventDisableTiming));
  VPG_CUDA(cudaEventCreateWithFlags(&b_done, cudaEventDisableTiming));

  for (int c = 0; c < n_cls; ++c) {
    const ClassPlan& p = plan[c];
    const int m = int(p.m);
    const int32_t* rows_p = rows.get();
    int32_t* assign_c = assign_all + p.row_off;
    GridParams gp = make_grid(p);

    // device: cell keys of the points and their sort, independent of the
    // center draw, overlap the host RNG
    int end_bits = 64;
    if (gp.packed) end_bits = packed_key_bits(gp);
    PointCells pc{};
    if (m > 1) pc = sort_points_by_cell(rows_p, p.row_off, p.n, rec.pos, gp, scalars.get() + 1, "", s);
    int32_t* pids_sorted = pc.pids_sorted;
    int32_t* run_start = pc.run_start;
    int32_t* run_len = pc.run_len;

    // m centers = Generator.choice(n, m) (clustering.py:51)
    DBuf<int32_t> d_local(m, s);
    if (p.n > 10000 && p.m > p.n / 50) {
      // tail shuffle: the host draws the swap targets (sequential stream),
      // the device resolves the swaps
      const int64_t stop = (p.n - p.m) > 1 ? (p.n - p.m) : 1;
      const int64_t steps = p.n - stop;
      int32_t* d_target = scratch_of<int32_t>(s, "swap_target", steps + 1);
      unsigned long long* d_keys = scratch_of<unsigned long long>(s, "swap_keys", steps + 1);
      unsigned long long* d_sk = scratch_of<unsigned long long>(s, "swap_sorted", steps + 1);
      int32_t* d_prev = scratch_of<int32_t>(s, "swap_prev", steps + 1);
      if (spec.targets && n_cls == 1 && spec.steps == steps) {
        // the speculative draw is this one: copy it as the thread writes it
        spec.adopted = true;
        VPG_LAUNCH(k_copy_when_ready, 64, 256, 0, s,
                   reinterpret_cast<const uint32_t*>(spec.targets->get()), spec.ready->get(),
                   reinterpret_cast<uint32_t*>(d_target), steps);
      } else {
        rng_ready();
        auto t = std::make_unique<HostBuf<int32_t>>(size_t(steps) + 1);
        for (int64_t k = 0; k < steps; ++k) (*t)[k] = int32_t(rng.bounded(uint64_t(p.n - 1 - k)));
        up.pinned(d_target, t->get(), size_t(steps), s);
        up_hold.push_back(std::move(t));
      }
      VPG_LAUNCH(k_swap_keys, grid_for(steps, block), block, 0, s, d_target, steps, d_keys);
      // by position only (bits 32..): the sort is stable and the keys arrive in
      // step order, so equal positions stay in step order
      const int pos_bits = bits_for(uint64_t(p.n > 1 ? p.n - 1 : 1));
      cub_call([&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortKeys(t, b, d_keys, d_sk, int(steps), 32, 32 + pos_bits, s);
      }, s);
      VPG_LAUNCH(k_swap_links, grid_for(steps, block), block, 0, s, d_sk, steps, p.n, d_prev);
      VPG_LAUNCH(k_swap_resolve, grid_for(steps, block), block, 0, s, d_target, d_sk, d_prev, steps,
                 p.n, p.m, d_local.get());
    } else {
      rng_ready();
      HostBuf<int64_t> picks(m);
      HostBuf<int32_t> picks32(m);
      rng_choice(rng, p.n, p.m, picks.get());
      for (int j = 0; j < m; ++j) picks32[j] = int32_t(picks[j]);
      up.pinned(d_local.get(), picks32.get(), size_t(m), s);
      VPG_CUDA(cudaStreamSynchronize(s));
    }
    clk.mark(1);

    DBuf<double> cpos(size_t(m) * 3, s);
    DBuf<unsigned long long> keys(m, s), skeys(m, s);
    DBuf<int32_t> ids(m, s), sids(m, s);
    DBuf<double4> spos(m, s);
    if (m == 1) {
      // a single center takes every point (clustering.py:100-101)
      gp.cell = 1.0;
      gp.packed = 1;
      VPG_LAUNCH(k_center_setup, 1, 32, 0, s, d_local.get(), m, rows_p, p.row_off, rec.pos, gp,
                 cpos.get(), crec_all.get() + p.center_off, keys.get(), ids.get());
      VPG_CUDA(cudaMemsetAsync(assign_c, 0, sizeof(int32_t) * p.n, s));
    } else {
      DBuf<CellEntry> table;
      DBuf<int2> dense;
      const bool use_dense = dense_cells_ok(gp, m);
      if (use_dense) {
        dense.alloc(size_t(dense_cells(gp)), s);
        VPG_CUDA(cudaMemsetAsync(dense.get(), 0, dense.bytes(), s));
      } else {
        table.alloc(gp.table_mask + 1, s);
        VPG_CUDA(cudaMemsetAsync(table.get(), 0xFF, table.bytes(), s));
      }
      const CellIndex cidx{table.get(), use_dense ? dense.get() : nullptr, gp.table_mask};
      VPG_LAUNCH(k_center_setup, grid_for(m, block), block, 0, s, d_local.get(), m, rows_p,
                 p.row_off, rec.pos, gp, cpos.get(), crec_all.get() + p.center_off, keys.get(),
                 ids.get());
      cub_call([&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, keys.get(), skeys.get(), ids.get(),
                                               sids.get(), m, 0, end_bits, s);
      }, s);
      VPG_LAUNCH(k_center_table, grid_for(m, block), block, 0, s, skeys.get(), sids.get(),
                 cpos.get(), m, gp, spos.get(), use_dense ? nullptr : table.get());
      if (use_dense)
        VPG_LAUNCH(k_center_dense, grid_for(m, block), block, 0, s, skeys.get(), m, dense.get());
      else
        VPG_LAUNCH(k_center_table_ends, grid_for(m, block), block, 0, s, skeys.get(), m, gp,
                   table.get());
      // part A layout order (the table no longer needs skeys/sids)
      VPG_LAUNCH(k_center_morton, grid_for(m, block), block, 0, s, cpos.get(), m, gp, keys.get(),
                 ids.get());
      // Morton bits: cell coordinates are clamped to [0, 2^21) per axis
      long long max_dim = 1;
      for (int a = 0; a < 3; ++a) max_dim = std::max(max_dim, gp.dims[a]);
      const int morton_bits = 3 * std::min(21, bits_for(uint64_t(max_dim)));
      cub_call([&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, keys.get(), skeys.get(), ids.get(),
                                               sids.get(), m, 0, morton_bits, s);
      }, s);
      VPG_CUDA(cudaMemsetAsync(scalars.get(), 0, sizeof(int32_t), s));
      ensure_dynamic_smem(reinterpret_cast<const void*>(k_assign_cells), kAssignSmem);
      VPG_LAUNCH(k_assign_cells, sm_count() * VPG_ASSIGN_MINB, kAssignWarps * 32, kAssignSmem, s, rows_p, p.row_off,
                 rec.pos, gp, cidx, spos.get(), pids_sorted, int(pc.oct_in_ids), run_start, run_len,
                 scalars.get() + 1, assign_c, fb_list, scalars.get());
      int32_t* far_list = scratch_of<int32_t>(s, "far_list", p.n + 1);
      auto* far_d = scratch_of<unsigned long long>(s, "far_d", p.n + 1);
      int32_t* far_j = scratch_of<int32_t>(s, "far_j", p.n + 1);
      VPG_CUDA(cudaMemsetAsync(far_count.get(), 0, sizeof(int32_t), s));
      VPG_LAUNCH(k_assign_fallback, sm_count() * 8, 256, 0, s, rows_p, p.row_off, rec.pos, gp,
                 cidx, spos.get(), fb_list, scalars.get(), assign_c, far_list,
                 far_count.get(), far_d, far_j);
      // points beyond the shell budget: tiled exact scan (grid sized for the
      // worst case; blocks past the list's end exit at once)
      for (int pass = 0; pass < 2; ++pass)
        VPG_LAUNCH(k_far_tiles, sm_count() * 4, 256, 0, s, rows_p, p.row_off, rec.pos, spos.get(),
                   m, far_list, far_count.get(), far_d, far_j, pass);
      VPG_LAUNCH(k_far_store, sm_count() * 2, 256, 0, s, far_list, far_count.get(), far_j,
                 assign_c);
    }
    clk.mark(2);

    // groups: stable sort of this class's records by center (clustering.py:55)
    VPG_LAUNCH(k_group_values, grid_for(p.n, block), block, 0, s, rows_p, p.row_off, p.n,
               values + p.row_off);
    int32_t* counts_c = counts_all.get() + p.center_off;
    int32_t* gstart_c = gstart_all.get() + p.center_off;
    {
      int32_t* sorted_keys = scratch_of<int32_t>(s, "sorted_keys", p.n);
      const int end_bit = bits_for(uint64_t(m > 1 ? m - 1 : 1));
      const int64_t nn = p.n;
      cub_call([&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, reinterpret_cast<uint32_t*>(assign_c),
                                               reinterpret_cast<uint32_t*>(sorted_keys),
                                               values + p.row_off, grp_rec + p.row_off, int(nn), 0,
                                               end_bit, s);
      }, s);
    }
    VPG_LAUNCH(k_histogram, grid_for(p.n, block, 1 << 30), block, 0, s, assign_c, p.n, counts_c);
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(t, b, counts_c, gstart_c, m, s);
    }, s);
    // oversize groups (> 2K members), in ascending group order
    DBuf<int32_t> over(m, s);
    DBuf<int64_t> over_info(size_t(m) * 4, s);
    {
      cub::CountingInputIterator<int32_t> it(0);
      Oversize pred{counts_c, int32_t(max_size)};
      cub_call([&](void* t, size_t& b) {
        return cub::DeviceSelect::If(t, b, it, over.get(), scalars.get() + 2, m, pred, s);
      }, s);
    }
    VPG_LAUNCH(k_oversize_info, grid_for(m, block), block, 0, s, over.get(), scalars.get() + 2,
               counts_c, gstart_c, crec_all.get() + p.center_off, over_info.get());
    int64_t* over_dst = scratch_of<int64_t>(s, "over_dst", size_t(m) + 1);
    int64_t* over_seg = scratch_of<int64_t>(s, "over_seg", size_t(m) * 3 + 3);
    {
      cub::CountingInputIterator<int32_t> it0(0);
      cub::TransformInputIterator<int64_t, OverCount, cub::CountingInputIterator<int32_t>> cnt_it(
          it0, OverCount{over_info.get()});
      // scanning all m entries is cheap; entries past n_over are unused
      cub_call([&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveSum(t, b, cnt_it, over_dst, m, s);
      }, s);
    }
    VPG_LAUNCH(k_oversize_seg, grid_for(m, block), block, 0, s, over_info.get(), scalars.get() + 2,
               over_dst, p.row_off, over_seg, scalars.get());
    int64_t* mask_off = scratch_of<int64_t>(s, "mask_off", size_t(m) + 1);
    {
      cub::CountingInputIterator<int32_t> it0(0);
      cub::TransformInputIterator<int64_t, MaskWords, cub::CountingInputIterator<int32_t>> mw_it(
          it0, MaskWords{over_info.get(), scalars.get() + 2});
      cub_call([&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveSum(t, b, mw_it, mask_off, m, s);
      }, s);
      VPG_LAUNCH(k_mask_total, 1, 1, 0, s, mask_off, over_info.get(), scalars.get() + 2, over_seg,
                 mask_total.get());
    }

    // ---- part A of this class: layout (device)
    {
      LayoutAcc* pre = scratch_of<LayoutAcc>(s, "layout_pre", size_t(m) + 1);
      LayoutAcc* pre_o = scratch_of<LayoutAcc>(s, "layout_pre_o", size_t(m) + 1);
      cub::TransformInputIterator<LayoutAcc, LayoutOf, const int32_t*> it(
          counts_c, LayoutOf{int32_t(max_size)});
      cub_call([&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveScan(t, b, it, pre, LayoutSum(), LayoutAcc{0, 0, 0, 0}, m, s);
      }, s);
      const int32_t* order = m > 1 ? sids.get() : ids.get();
      cub::CountingInputIterator<int32_t> ci(0);
      cub::TransformInputIterator<LayoutAcc, LayoutOfPerm, cub::CountingInputIterator<int32_t>> ito(
          ci, LayoutOfPerm{counts_c, order, int32_t(max_size)});
      cub_call([&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveScan(t, b, ito, pre_o, LayoutSum(), LayoutAcc{0, 0, 0, 0}, m,
                                              s);
      }, s);
      VPG_LAUNCH(k_layout_a, grid_for(m, block), block, 0, s, counts_c, gstart_c,
                 crec_all.get() + p.center_off, pre, order, pre_o, m, int32_t(max_size), p.row_off,
                 appended_before, acc.get(), g->cl_off.get(), g->cl_size.get(), g->w_off.get(),
                 a_src.get(), g->cl_center.get(), g->ref_of.get(),
                 ne_prefix_all.get() + p.center_off);
      VPG_LAUNCH(k_layout_a_totals, 1, 1, 0, s, counts_c, pre, m, int32_t(max_size),
                 appended_before, acc.get(), cls_info.get() + 4 * c);
      VPG_CUDA(cudaMemcpyAsync(ranges.get() + 2 * c, cls_info.get() + 4 * c, 2 * sizeof(int64_t),
                               cudaMemcpyDeviceToDevice, s));
      if (c == n_cls - 1) {
        VPG_CUDA(cudaMemcpyAsync(h_acc.get(), acc.get(), 8 * sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, s));
        count_transfer(0, 64);
        VPG_CUDA(cudaEventRecord(acc_ready, s));
      }
    }
    // sizes of the oversize staging (nothing heavy is queued before this sync)
    HostBuf<int32_t> h_scalars(4);
    HostBuf<int64_t> h_mask_total(1 + 3 * (kBulkPieces + 1));
    VPG_CUDA(cudaMemcpyAsync(h_scalars.get(), scalars.get(), 4 * sizeof(int32_t),
                             cudaMemcpyDeviceToHost, s));
    VPG_CUDA(cudaMemcpyAsync(h_mask_total.get(), mask_total.get(),
                             sizeof(int64_t) * (1 + 3 * (kBulkPieces + 1)), cudaMemcpyDeviceToHost, s));
    count_transfer(0, 16 + 8 * (1 + 3 * (kBulkPieces + 1)));
    // the staging below runs on the side stream from here; part A goes on s
    // now, before the host learns the staging sizes
    cudaStream_t side = side_stream();
    cudaEvent_t sized;
    VPG_CUDA(cudaEventCreateWithFlags(&sized, cudaEventDisableTiming));
    VPG_CUDA(cudaEventRecord(sized, s));
    VPG_CUDA(cudaStreamWaitEvent(side, sized, 0));
    // ---- part A of this class: permutation, pack, aggregate (device, async)
    VPG_LAUNCH(k_fill_perm, sm_count() * 8, 256, 0, s, ranges.get() + 2 * c, g->cl_off.get(),
               g->cl_size.get(), a_src.get(), g->ref_of.get(), grp_rec, nullptr, g->perm.get(),
               g->clpos.get(), static_cast<int32_t*>(nullptr));
    // part B (split results) may start once this class's rows are placed
    VPG_CUDA(cudaEventRecord(placed, s));
    if (with_ops) {
      // the operator fields may still be in flight (async upload): the
      // clustering above only needed pos, kind and class_id
      if (fields_ready && c == 0) VPG_CUDA(cudaStreamWaitEvent(s, fields_ready, 0));
      pack_members(g, rec, rows_p ? rows_p + p.row_off : nullptr, p.n, p.row_off, members, s);
      aggregate_range(g, members, ranges.get() + 2 * c, m, S, s);
      // children in earlier classes were packed before these parents existed
      if (c > 0 && rows_p) link_children(g, rec, rows_p + p.row_off, p.n, s);
    }
    DebugClock dstage(s);
    VPG_CUDA(cudaEventSynchronize(sized));
    cudaEventDestroy(sized);
    dstage.mark("stage: sizes known", false);
    g->info.n_fallback += h_scalars[0];
    const int n_over = h_scalars[2];
    const int64_t staged = n_over > 0 ? h_scalars[3] : 0;
    // oversize members and positions to the host, queued ahead of part A
    HostBuf<int64_t> info(size_t(n_over) * 4 + 4);
    auto h_srec_own = std::make_unique<HostBuf<int32_t>>(size_t(staged) + 1);
    HostBuf<int32_t>& h_srec = *h_srec_own;
    HostBuf<int32_t> h_slot(size_t(n_over) + 1);
    HostBuf<double> h_xyzd(size_t(staged) * 4 + 4);  // x | y | z | d0
    const int64_t n_mask = n_over > 0 ? h_mask_total[0] : 0;
    HostBuf<unsigned long long> h_masks(size_t(n_mask) + 1);
    HostBuf<int32_t> h_moved(size_t(staged) + 1);
    // kept until part B applies the deferred first splits
    auto d_masks_own = std::make_unique<DBuf<unsigned long long>>(size_t(n_mask) + 1, side);
    d_masks_own->s = s;  // released on s, which joins part B (its last reader)
    cudaEvent_t staged_ready;
    VPG_CUDA(cudaEventCreateWithFlags(&staged_ready, cudaEventDisableTiming));
    // positions, distances and mask rows go in pieces, last groups first (the
    // split loop pops them first); piece_ready[j] closes piece j
    std::vector<cudaEvent_t> piece_ready(n_over > 0 ? kBulkPieces : 0);
    const int64_t* bounds = h_mask_total.get() + 1;
    if (n_over > 0) {
      int32_t* d_srec = scratch_of<int32_t>(s, "staged_rec", size_t(staged) + 1);
      int32_t* d_slot = scratch_of<int32_t>(s, "staged_slot", size_t(n_over) + 1);
      double* d_xyzd = scratch_of<double>(s, "staged_xyzd", size_t(staged) * 4 + 4);
      unsigned long long* d_masks = d_masks_own->get();
      int32_t* d_moved = scratch_of<int32_t>(s, "first_moved", size_t(staged) + 1);
      VPG_CUDA(cudaMemsetAsync(d_moved, 0, sizeof(int32_t) * staged, side));
      VPG_CUDA(cudaMemsetAsync(d_slot, 0x7F, sizeof(int32_t) * n_over, side));
      VPG_LAUNCH(k_gather_oversize, std::min<int64_t>(n_over, 65535), 128, 0, side, grp_rec, over_seg,
                 scalars.get() + 2, over_info.get(), rec.pos, d_srec, d_xyzd, d_xyzd + staged,
                 d_xyzd + 2 * staged, d_xyzd + 3 * staged, d_slot);
      VPG_LAUNCH(k_first_split_masks, std::min<int64_t>(n_over, 65535), 256, 0, side, over_seg,
                 scalars.get() + 2, mask_off, d_xyzd, d_xyzd + staged, d_xyzd + 2 * staged,
                 d_xyzd + 3 * staged, d_masks, d_moved);
      dstage.mark("stage: kernels queued", false);
      // the staging goes to the host from the side stream, beside part A
      VPG_CUDA(cudaMemcpyAsync(info.get(), over_info.get(), sizeof(int64_t) * 4 * n_over,
                               cudaMemcpyDeviceToHost, side));
      VPG_CUDA(cudaMemcpyAsync(h_srec.get(), d_srec, sizeof(int32_t) * staged,
                               cudaMemcpyDeviceToHost, side));
      VPG_CUDA(cudaMemcpyAsync(h_slot.get(), d_slot, sizeof(int32_t) * n_over,
                               cudaMemcpyDeviceToHost, side));
      VPG_CUDA(cudaMemcpyAsync(h_moved.get(), d_moved, sizeof(int32_t) * staged,
                               cudaMemcpyDeviceToHost, side));
      VPG_CUDA(cudaEventRecord(staged_ready, side));
      for (int j = kBulkPieces - 1; j >= 0; --j) {
        const int64_t s0 = bounds[3 * j + 1], s1 = bounds[3 * j + 4];
        const int64_t k0 = bounds[3 * j + 2], k1 = bounds[3 * j + 5];
        if (s1 > s0)
          for (int a = 0; a < 4; ++a)
            VPG_CUDA(cudaMemcpyAsync(h_xyzd.get() + a * staged + s0, d_xyzd + a * staged + s0,
                                     sizeof(double) * (s1 - s0), cudaMemcpyDeviceToHost, side));
        if (k1 > k0)
          VPG_CUDA(cudaMemcpyAsync(h_masks.get() + k0, d_masks + k0,
                                   sizeof(unsigned long long) * (k1 - k0), cudaMemcpyDeviceToHost,
                                   side));
        VPG_CUDA(cudaEventCreateWithFlags(&piece_ready[j], cudaEventDisableTiming));
        VPG_CUDA(cudaEventRecord(piece_ready[j], side));
      }
      count_transfer(0, 36 * n_over + 40 * staged + 8 * n_mask);
    } else {
      VPG_CUDA(cudaEventRecord(staged_ready, side));
    }
    clk.mark(3);

    // ---- split loop on the oversize groups (host, exact RNG order), while
    // the device aggregates part A
    DebugClock dbg(s);
    VPG_CUDA(cudaEventSynchronize(staged_ready));
    cudaEventDestroy(staged_ready);
    int64_t appended_c = 0;
    if (n_over > 0) {
      dbg.mark("split: info+gather+D2H", false);
      std::vector<SplitGroup> groups(n_over);
      std::vector<int64_t> cslot(n_over);
      int64_t b = 0;
      for (int k = 0; k < n_over; ++k) {
        const int64_t cnt = info[k * 4 + 1];
        groups[k] = SplitGroup{b, cnt, int32_t(info[k * 4 + 3])};
        cslot[k] = h_slot[k] < staged ? int64_t(h_slot[k]) : -1;
        b += cnt;
      }
      g->info.n_staged += staged;
      dbg.mark("split: groups", false);
      double* xyzd = h_xyzd.get();
      SplitStats st;
      std::vector<DeferredSplit> deferred;
      // the bulk piece holding original group k, waited for on first use
      int waited_from = kBulkPieces;
      const std::function<void(int64_t)> need_bulk = [&](int64_t k) {
        int j = kBulkPieces - 1;
        while (j > 0 && bounds[3 * j] > k) --j;
        while (waited_from > j) {
          --waited_from;
          VPG_CUDA(cudaEventSynchronize(piece_ready[waited_from]));
        }
      };
      rng_ready();
      n_splits += split_oversize_soa(
          rng, SplitMembers{h_srec.get(), xyzd, xyzd + staged, xyzd + 2 * staged, xyzd + 3 * staged},
          groups, cslot, max_size, &g->info.split_visits, h_masks.get(), dbg.on ? &st : nullptr,
          h_moved.get(), 2 * max_size <= 3 * kApplyThreads ? &deferred : nullptr, &need_bulk);
      for (int j = 0; j < kBulkPieces; ++j) {
        VPG_CUDA(cudaEventSynchronize(piece_ready[j]));  // host buffers outlive no copy
        cudaEventDestroy(piece_ready[j]);
      }
      dbg.mark("split: loop", false);
      if (dbg.on) {
        fprintf(stderr, "[vpg] class %d: %lld oversize groups, %lld staged members, %lld groups after\n",
                c, (long long)n_over, (long long)staged, (long long)groups.size());
        const char* kinds[3] = {"first split, final", "first split, again", "later split"};
        for (int q = 0; q < 3; ++q)
          fprintf(stderr, "[vpg]   %-20s %6lld splits %8lld members %8.3f ms\n", kinds[q],
                  (long long)st.n[q], (long long)st.members[q], st.ns[q] * 1e-6);
      }
      const int64_t base_split = split_total;
      auto hb_own = std::make_unique<HostBuf<int64_t>>(groups.size() * 8 + 8);
      int64_t* hb = hb_own->get();
      for (size_t k = 0; k < groups.size(); ++k) {
        const int64_t sz = groups[k].size;
        const int64_t j = k < size_t(n_over) ? info[k * 4] : -1 - (int64_t(k) - n_over);
        const int64_t e[8] = {c, j, sz, rows_b, w_b, base_split + groups[k].begin,
                              groups[k].center, 0};
        std::memcpy(hb + 8 * k, e, sizeof(e));
        rows_b += sz;
        w_b += (sz * sz + 3) & ~int64_t(3);
      }
      auto hd_own = std::make_unique<HostBuf<int64_t>>(deferred.size() * 3 + 3);
      for (size_t k = 0; k < deferred.size(); ++k) {
        hd_own->get()[3 * k] = deferred[k].begin;
        hd_own->get()[3 * k + 1] = deferred[k].size;
        hd_own->get()[3 * k + 2] = deferred[k].row;
      }
      chunks.push_back(SplitChunk{std::move(h_srec_own), staged, std::move(hb_own),
                                  int64_t(groups.size()), std::move(hd_own),
                                  int64_t(deferred.size()), std::move(d_masks_own)});
      split_total += staged;
      nb_total += int64_t(groups.size());
      appended_c = int64_t(groups.size()) - n_over;
      dbg.mark("split: mods", false);
    }
    appended_before += appended_c;
    clk.mark(4);
  }
  g->info.n_splits = n_splits;
  rng_ready();
  rng.store(rng_state);

  // ---- part B: the split results, appended after part A
  VPG_CUDA(cudaEventSynchronize(acc_ready));
  cudaEventDestroy(acc_ready);
  const int64_t m_a = h_acc[0];
  const int64_t nb = nb_total;
  const int64_t M = m_a + nb;
  g->m = M;
  // Part B runs on a second stream, concurrently with part A's pack and
  // aggregate (still running on s): it only needs part A's placement (the
  // `placed` event) and writes disjoint rows.  Its buffers are allocated on sb
  // and handed to s for their release; s joins sb before anything reads them.
  cudaStream_t sb = side_stream(1);
  VPG_CUDA(cudaStreamWaitEvent(sb, placed, 0));
  if (with_ops && fields_ready) VPG_CUDA(cudaStreamWaitEvent(sb, fields_ready, 0));
  {
    // final cluster arrays: part A copied over, part B written below (the
    // old part A arrays are freed on s, after part A's aggregate)
    DBuf<int32_t> f_off(M + 1, sb), f_size(M + 1, sb), f_center(M + 1, sb), f_ref(M + 1, sb);
    DBuf<int64_t> f_w(M + 1, sb), f_src(M + 1, sb);
    auto copy_a = [&](void* dst, const void* src, size_t elem) {
      if (m_a) VPG_CUDA(cudaMemcpyAsync(dst, src, elem * m_a, cudaMemcpyDeviceToDevice, sb));
    };
    copy_a(f_off.get(), g->cl_off.get(), 4);
    copy_a(f_size.get(), g->cl_size.get(), 4);
    copy_a(f_center.get(), g->cl_center.get(), 4);
    copy_a(f_ref.get(), g->ref_of.get(), 4);
    copy_a(f_w.get(), g->w_off.get(), 8);
    copy_a(f_src.get(), a_src.get(), 8);
    for (auto* b : {&f_off, &f_size, &f_center, &f_ref}) b->s = s;
    for (auto* b : {&f_w, &f_src}) b->s = s;
    // the old arrays are released on s: only after sb has copied them
    cudaEvent_t copied;
    VPG_CUDA(cudaEventCreateWithFlags(&copied, cudaEventDisableTiming));
    VPG_CUDA(cudaEventRecord(copied, sb));
    VPG_CUDA(cudaStreamWaitEvent(s, copied, 0));
    cudaEventDestroy(copied);
    g->cl_off = std::move(f_off);
    g->cl_size = std::move(f_size);
    g->cl_center = std::move(f_center);
    g->ref_of = std::move(f_ref);
    g->w_off = std::move(f_w);
    a_src = std::move(f_src);
  }
  DBuf<int64_t> d_b(size_t(nb) * 8 + 8, sb);
  DBuf<int32_t> d_split(size_t(split_total) + 1, sb);
  // link_children reads d_split on s after part B: free it on s (s waits
  // for b_done, so every use on sb precedes the free in s's order)
  d_split.s = s;
  DBuf<int64_t> range_b(2, sb);
  if (nb) {
    int64_t ob = 0, os = 0;
    for (const SplitChunk& ch : chunks) {
      up.pinned(d_b.get() + ob, ch.b->get(), size_t(ch.n_b) * 8, sb);
      up.pinned(d_split.get() + os, ch.rec->get(), size_t(ch.n_rec), sb);
      if (ch.n_deferred) {
        int64_t* d_def = scratch_of<int64_t>(sb, "deferred_splits", size_t(ch.n_deferred) * 3);
        up.pinned(d_def, ch.deferred->get(), size_t(ch.n_deferred) * 3, sb);
        VPG_LAUNCH(k_apply_first_splits, int(std::min<int64_t>(ch.n_deferred, 65535)),
                   kApplyThreads, 0, sb, d_def, ch.n_deferred, ch.masks->get(),
                   d_split.get() + os);
      }
      ob += ch.n_b * 8;
      os += ch.n_rec;
    }
    VPG_LAUNCH(k_layout_b, grid_for(nb, block), block, 0, sb, d_b.get(), nb, acc.get(),
               cls_info.get(), ne_prefix_all.get(), class_center_off.get(), g->cl_off.get(),
               g->cl_size.get(), g->w_off.get(), a_src.get(), g->cl_center.get(), g->ref_of.get());
  }
  VPG_LAUNCH(k_layout_close, 1, 1, 0, sb, nb, rows_b, w_b, acc.get(), g->cl_off.get(),
             g->w_off.get(), range_b.get());
  if (nb) {
    VPG_LAUNCH(k_fill_perm, sm_count() * 8, 256, 0, sb, range_b.get(), g->cl_off.get(),
               g->cl_size.get(), a_src.get(), g->ref_of.get(), grp_rec, d_split.get(),
               g->perm.get(), g->clpos.get(), static_cast<int32_t*>(nullptr));
    if (with_ops) {
      pack_members(g, rec, d_split.get(), split_total, 0, members, sb);
      aggregate_range(g, members, range_b.get(), nb, S, sb);
    }
  }
  VPG_CUDA(cudaEventRecord(b_done, sb));
  VPG_CUDA(cudaStreamWaitEvent(s, b_done, 0));
  cudaEventDestroy(placed);
  cudaEventDestroy(b_done);
  // children in part A of the split results' records: after part A's
  // aggregate wrote those rows (stream order on s)
  if (with_ops && nb) link_children(g, rec, d_split.get(), split_total, s);
  g->internal_of.alloc(M + 1, s);
  VPG_LAUNCH(k_invert_ref, grid_for(M, block), block, 0, s, g->ref_of.get(), M,
             g->internal_of.get());
  // totals: nnz (sum of s^2) and the padded kernel length, to pinned memory
  // without waiting (vpg_graph::sync_totals); the staging needs only the
  // bound on the cluster size (every cluster has at most 2K members)
  g->tot_host.alloc(2);
  {
    int64_t* d_tot = scratch_of<int64_t>(s, "nnz_total", 2);
    cub::TransformInputIterator<int64_t, SquareOp, const int32_t*> sq_it(g->cl_size.get(), SquareOp());
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceReduce::Sum(t, b, sq_it, d_tot, int(M), s);
    }, s);
    VPG_CUDA(cudaMemcpyAsync(d_tot + 1, g->w_off.get() + M, sizeof(int64_t),
                             cudaMemcpyDeviceToDevice, s));
    VPG_CUDA(cudaMemcpyAsync(g->tot_host.get(), d_tot, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost,
                             s));
    count_transfer(0, 16);
  }
  g->max_cluster = int32_t(std::min<int64_t>(max_size, std::max<int64_t>(n, 1)));
  if (with_ops && fields_ready) VPG_CUDA(cudaStreamWaitEvent(s, fields_ready, 0));
  if (with_ops) finalize_operators_async(g, rec, s, nullptr, true);
  clk.mark(5);
  if (with_ops) finalize_chunks(g, s);
  // pinned inputs part B's kernels read from the host stay with the graph
  for (SplitChunk& ch : chunks) {
    g->hold_host(std::move(ch.rec));
    g->hold_host(std::move(ch.b));
    g->hold_host(std::move(ch.deferred));
  }
  for (auto& k : up.keep) g->hold_host(std::move(k));
  for (auto& b : up_hold) g->hold_host(std::move(b));
  rng_ready();
  g->hold_host(std::move(spec.targets));
  g->hold_host(std::move(spec.ready));
  up.keep.clear();
  VPG_CUDA(cudaEventCreateWithFlags(&g->done_ev, cudaEventDisableTiming));
  VPG_CUDA(cudaEventRecord(g->done_ev, s));
  g->tot_pending = true;
  clk.mark(6);
}

// The split loop over oversize groups whose members are on the device (SoA x,
// y, z, d0 and the member ids, groups back to back): the first splits' bit
// rows and moved counts are computed on the device, the loop runs on the host
// with the deferred-first-split fast path, and the deferred partitions are
// applied to the device ids -- the sharded build's equivalent of the build's
// own split stage.  ids (device) end in final member order.
void split_groups_device(vpg_pcg64* state, int32_t* d_ids, const double* d_x, const double* d_y,
                         const double* d_z, const double* d_d0, int64_t n_groups,
                         const int64_t* sizes, const int64_t* centers, const int64_t* cslot_in,
                         int64_t max_size, std::vector<SplitGroup>& groups, int64_t* n_splits,
                         cudaStream_t s) {
  Pcg64 rng(*state);
  groups.assign(static_cast<size_t>(n_groups), SplitGroup{0, 0, 0});
  std::vector<int64_t> cslot(static_cast<size_t>(n_groups));
  std::vector<int64_t> seg(static_cast<size_t>(n_groups) * 3 + 3), moff(static_cast<size_t>(n_groups) + 1);
  int64_t total = 0, words = 0;
  for (int64_t k = 0; k < n_groups; ++k) {
    groups[k] = SplitGroup{total, sizes[k], centers[k]};
    cslot[k] = cslot_in[k];
    seg[3 * k] = 0;
    seg[3 * k + 1] = sizes[k];
    seg[3 * k + 2] = total;
    moff[k] = words;
    words += sizes[k] * ((sizes[k] + 63) / 64);
    total += sizes[k];
  }
  *n_splits = 0;
  if (n_groups == 0) {
    rng.store(state);
    return;
  }
  HostUpload up;
  DBuf<int64_t> d_seg(seg.size(), s), d_moff(moff.size(), s);
  DBuf<int32_t> d_n(1, s), d_moved(static_cast<size_t>(total) + 1, s);
  DBuf<unsigned long long> d_masks(static_cast<size_t>(words) + 1, s);
  up.put(d_seg.get(), seg.data(), seg.size(), s);
  up.put(d_moff.get(), moff.data(), moff.size(), s);
  const int32_t ng32 = int32_t(n_groups);
  up.put(d_n.get(), &ng32, 1, s);
  VPG_CUDA(cudaMemsetAsync(d_moved.get(), 0, sizeof(int32_t) * total, s));
  VPG_LAUNCH(k_first_split_masks, int(std::min<int64_t>(n_groups, 65535)), 256, 0, s, d_seg.get(),
             d_n.get(), d_moff.get(), d_x, d_y, d_z, d_d0, d_masks.get(), d_moved.get());
  HostBuf<int32_t> h_ids(static_cast<size_t>(total) + 1), h_moved(static_cast<size_t>(total) + 1);
  HostBuf<double> h_xyzd(static_cast<size_t>(total) * 4 + 4);
  HostBuf<unsigned long long> h_masks(static_cast<size_t>(words) + 1);
  VPG_CUDA(cudaMemcpyAsync(h_ids.get(), d_ids, sizeof(int32_t) * total, cudaMemcpyDeviceToHost, s));
  const double* src[4] = {d_x, d_y, d_z, d_d0};
  for (int a = 0; a < 4; ++a)
    VPG_CUDA(cudaMemcpyAsync(h_xyzd.get() + a * total, src[a], sizeof(double) * total,
                             cudaMemcpyDeviceToHost, s));
  VPG_CUDA(cudaMemcpyAsync(h_masks.get(), d_masks.get(), sizeof(unsigned long long) * words,
                           cudaMemcpyDeviceToHost, s));
  VPG_CUDA(cudaMemcpyAsync(h_moved.get(), d_moved.get(), sizeof(int32_t) * total,
                           cudaMemcpyDeviceToHost, s));
  VPG_CUDA(cudaStreamSynchronize(s));
  std::vector<DeferredSplit> deferred;
  double* xyzd = h_xyzd.get();
  int64_t visits = 0;
  *n_splits = split_oversize_soa(
      rng, SplitMembers{h_ids.get(), xyzd, xyzd + total, xyzd + 2 * total, xyzd + 3 * total},
      groups, cslot, max_size, &visits, h_masks.get(), nullptr, h_moved.get(),
      2 * max_size <= 3 * kApplyThreads ? &deferred : nullptr);
  // host order for the splits it made, then the deferred partitions on the device
  up.pinned(d_ids, h_ids.get(), static_cast<size_t>(total), s);
  if (!deferred.empty()) {
    HostBuf<int64_t> hd(deferred.size() * 3);
    for (size_t k = 0; k < deferred.size(); ++k) {
      hd[3 * k] = deferred[k].begin;
      hd[3 * k + 1] = deferred[k].size;
      hd[3 * k + 2] = deferred[k].row;
    }
    DBuf<int64_t> d_def(deferred.size() * 3, s);
    up.pinned(d_def.get(), hd.get(), deferred.size() * 3, s);
    VPG_LAUNCH(k_apply_first_splits, int(std::min<size_t>(deferred.size(), 65535)), kApplyThreads,
               0, s, d_def.get(), int64_t(deferred.size()), d_masks.get(), d_ids);
    VPG_CUDA(cudaStreamSynchronize(s));
  } else {
    VPG_CUDA(cudaStreamSynchronize(s));
  }
  // a deferred split's new center is the pick in the original order: the
  // host's ids for that range are still the original order, so it holds
  rng.store(state);
}

// Generator.choice(n, m, replace=False) with the picks left on the device
// (int32): the tail shuffle's targets are drawn on the host and its swaps
// resolved on the device as in the build; Floyd's branch (small m) on the
// host.  Synchronous on return (the host buffers are released).
void choice_device(vpg_pcg64* state, int64_t n, int64_t m, int32_t* d_out, cudaStream_t s) {
  VPG_REQUIRE(m >= 0 && m <= n && n < (int64_t(1) << 31), VPG_EINVAL,
              "Cannot take a larger sample than population when replace is False");
  if (m == 0) return;
  Pcg64 rng(*state);
  const int block = 256;
  HostUpload up;
  if (n > 10000 && m > n / 50) {
    const int64_t stop = (n - m) > 1 ? (n - m) : 1;
    const int64_t steps = n - stop;
    HostBuf<int32_t> t(static_cast<size_t>(steps) + 1);
    for (int64_t k = 0; k < steps; ++k) t[k] = int32_t(rng.bounded(uint64_t(n - 1 - k)));
    DBuf<int32_t> d_target(size_t(steps) + 1, s), d_prev(size_t(steps) + 1, s);
    DBuf<unsigned long long> d_keys(size_t(steps) + 1, s), d_sk(size_t(steps) + 1, s);
    up.pinned(d_target.get(), t.get(), size_t(steps), s);
    VPG_LAUNCH(k_swap_keys, grid_for(steps, block), block, 0, s, d_target.get(), steps,
               d_keys.get());
    const int pos_bits = bits_for(uint64_t(n > 1 ? n - 1 : 1));
    cub_call([&](void* tmp, size_t& b) {
      return cub::DeviceRadixSort::SortKeys(tmp, b, d_keys.get(), d_sk.get(), int(steps), 32,
                                            32 + pos_bits, s);
    }, s);
    VPG_LAUNCH(k_swap_links, grid_for(steps, block), block, 0, s, d_sk.get(), steps, n,
               d_prev.get());
    VPG_LAUNCH(k_swap_resolve, grid_for(steps, block), block, 0, s, d_target.get(), d_sk.get(),
               d_prev.get(), steps, n, m, d_out);
    VPG_CUDA(cudaStreamSynchronize(s));
  } else {
    std::vector<int64_t> picks(static_cast<size_t>(m));
    rng_choice(rng, n, m, picks.data());
    HostBuf<int32_t> p32(static_cast<size_t>(m));
    for (int64_t j = 0; j < m; ++j) p32[j] = int32_t(picks[j]);
    up.pinned(d_out, p32.get(), size_t(m), s);
    VPG_CUDA(cudaStreamSynchronize(s));
  }
  rng.store(state);
}

// Exact nearest center (lowest index on ties) of every point against given
// centers -- the assignment step of clustering.py:96-148 on its own, for a
// shard's rows against the replicated centers of a class.  The result does
// not depend on the grid; lo/hi (the class bounding box) only size it like
// the single-device build.
int64_t assign_nearest(const double* pos, int64_t n, const double* cpos, int m, const double* lo,
                       const double* hi, int32_t* assign, cudaStream_t s) {
  if (n <= 0) return 0;
  VPG_REQUIRE(m >= 1, VPG_EINVAL, "no centers");
  if (m == 1) {  // a single center takes every point (clustering.py:100-101)
    VPG_CUDA(cudaMemsetAsync(assign, 0, sizeof(int32_t) * n, s));
    return 0;
  }
  const int block = 256;
  ClassPlan p{};
  p.n = n;
  p.m = m;
  for (int a = 0; a < 3; ++a) {
    p.lo[a] = lo[a];
    p.hi[a] = hi[a];
  }
  const GridParams gp = make_grid(p);
  DBuf<int32_t> scalars(4, s);
  DBuf<int32_t> far_count(1, s);
  VPG_CUDA(cudaMemsetAsync(scalars.get(), 0, scalars.bytes(), s));
  FbEntry* fb_list = scratch_of<FbEntry>(s, "an_fb_list", n + 1);
  const PointCells pc = sort_points_by_cell(nullptr, 0, n, pos, gp, scalars.get() + 1, "an_", s);
  DBuf<unsigned long long> keys(m, s), skeys(m, s);
  DBuf<int32_t> ids(m, s), sids(m, s);
  DBuf<double4> spos(m, s);
  DBuf<CellEntry> table;
  DBuf<int2> dense;
  const bool use_dense = dense_cells_ok(gp, m);
  if (use_dense) {
    dense.alloc(size_t(dense_cells(gp)), s);
    VPG_CUDA(cudaMemsetAsync(dense.get(), 0, dense.bytes(), s));
  } else {
    table.alloc(gp.table_mask + 1, s);
    VPG_CUDA(cudaMemsetAsync(table.get(), 0xFF, table.bytes(), s));
  }
  const CellIndex cidx{table.get(), use_dense ? dense.get() : nullptr, gp.table_mask};
  VPG_LAUNCH(k_center_keys, grid_for(m, block), block, 0, s, cpos, m, gp, keys.get(), ids.get());
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, keys.get(), skeys.get(), ids.get(), sids.get(), m,
                                           0, gp.packed ? packed_key_bits(gp) : 64, s);
  }, s);
  VPG_LAUNCH(k_center_table, grid_for(m, block), block, 0, s, skeys.get(), sids.get(), cpos, m, gp,
             spos.get(), use_dense ? nullptr : table.get());
  if (use_dense)
    VPG_LAUNCH(k_center_dense, grid_for(m, block), block, 0, s, skeys.get(), m, dense.get());
  else
    VPG_LAUNCH(k_center_table_ends, grid_for(m, block), block, 0, s, skeys.get(), m, gp,
               table.get());
  ensure_dynamic_smem(reinterpret_cast<const void*>(k_assign_cells), kAssignSmem);
  VPG_LAUNCH(k_assign_cells, sm_count() * VPG_ASSIGN_MINB, kAssignWarps * 32, kAssignSmem, s, nullptr, 0, pos, gp,
             cidx, spos.get(), pc.pids_sorted, int(pc.oct_in_ids), pc.run_start, pc.run_len,
             scalars.get() + 1, assign,
             fb_list, scalars.get());
  int32_t* far_list = scratch_of<int32_t>(s, "an_far_list", n + 1);
  auto* far_d = scratch_of<unsigned long long>(s, "an_far_d", n + 1);
  int32_t* far_j = scratch_of<int32_t>(s, "an_far_j", n + 1);
  VPG_CUDA(cudaMemsetAsync(far_count.get(), 0, sizeof(int32_t), s));
  VPG_LAUNCH(k_assign_fallback, sm_count() * 8, 256, 0, s, nullptr, 0, pos, gp, cidx,
             spos.get(), fb_list, scalars.get(), assign, far_list, far_count.get(), far_d, far_j);
  for (int pass = 0; pass < 2; ++pass)
    VPG_LAUNCH(k_far_tiles, sm_count() * 4, 256, 0, s, nullptr, 0, pos, spos.get(), m, far_list,
               far_count.get(), far_d, far_j, pass);
  VPG_LAUNCH(k_far_store, sm_count() * 2, 256, 0, s, far_list, far_count.get(), far_j, assign);
  int32_t h_fb = 0;
  VPG_CUDA(cudaMemcpyAsync(&h_fb, scalars.get(), sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  VPG_CUDA(cudaStreamSynchronize(s));
  count_transfer(0, 4);
  return h_fb;
}

}  // namespace vpg

// Host-side replica of numpy.random.Generator(PCG64) for the draws the
// reference's clustering makes, and the sequential split loop that consumes
// them.  Compiled with -ffp-contract=off: the split distances must round
// exactly like numpy's.
//
//   Generator.choice(n, m, replace=False)   clustering.py:51
//   Generator.integers(k)                   clustering.py:68
//   split loop                              clustering.py:58-85
//
// numpy (2.3.5 here) is a third-party dependency of the reference
// (pyproject.toml:11); its PCG64 stream and bounded-integer algorithms are
// restated from the published algorithm and pinned against numpy itself in
// tests/test_rng.py.
#pragma once
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/volpg_b200.h"

namespace vpg {

typedef unsigned __int128 u128;

struct Pcg64 {
  u128 state, inc;
  bool has32;
  uint32_t buf32;

  explicit Pcg64(const vpg_pcg64& s)
      : state((u128(s.state_hi) << 64) | s.state_lo),
        inc((u128(s.inc_hi) << 64) | s.inc_lo),
        has32(s.has_uint32 != 0),
        buf32(s.uinteger) {}

  void store(vpg_pcg64* s) const {
    s->state_hi = uint64_t(state >> 64);
    s->state_lo = uint64_t(state);
    s->inc_hi = uint64_t(inc >> 64);
    s->inc_lo = uint64_t(inc);
    s->has_uint32 = has32 ? 1 : 0;
    s->uinteger = buf32;  // numpy leaves the consumed half in place
  }

  // PCG XSL-RR 128/64: advance, then permute the new state.
  uint64_t next64() {
    static const u128 kMul = (u128(0x2360ED051FC65DA4ull) << 64) | 0x4385DF649FCCF645ull;
    state = state * kMul + inc;
    uint64_t x = uint64_t(state >> 64) ^ uint64_t(state);
    unsigned rot = unsigned(state >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }

  // numpy's next_uint32 keeps the unused upper half across calls.
  uint32_t next32() {
    if (has32) {
      has32 = false;
      return buf32;
    }
    uint64_t v = next64();
    has32 = true;
    buf32 = uint32_t(v >> 32);
    return uint32_t(v);
  }

  // Uniform integer in [0, rng] (numpy random_bounded_uint64, unmasked).
  uint64_t bounded(uint64_t rng) {
    if (rng == 0) return 0;
    if (rng <= 0xFFFFFFFFull) {
      if (rng == 0xFFFFFFFFull) return next32();
      const uint32_t r32 = uint32_t(rng);
      const uint32_t span = r32 + 1u;  // Lemire's nearly-divisionless method
      uint64_t prod = uint64_t(next32()) * span;
      uint32_t low = uint32_t(prod);
      if (low < span) {
        const uint32_t floor_ = (0xFFFFFFFFu - r32) % span;
        while (low < floor_) {
          prod = uint64_t(next32()) * span;
          low = uint32_t(prod);
        }
      }
      return prod >> 32;
    }
    if (rng == 0xFFFFFFFFFFFFFFFFull) return next64();
    const uint64_t span = rng + 1;
    u128 prod = u128(next64()) * span;
    uint64_t low = uint64_t(prod);
    if (low < span) {
      const uint64_t floor_ = (0xFFFFFFFFFFFFFFFFull - rng) % span;
      while (low < floor_) {
        prod = u128(next64()) * span;
        low = uint64_t(prod);
      }
    }
    return uint64_t(prod >> 64);
  }
};

// Open-addressing map int64 -> int64 for the sparse Fisher-Yates tail.
class SparseSwap {
 public:
  explicit SparseSwap(size_t expected) {
    size_t cap = 16;
    while (cap < expected * 2) cap <<= 1;
    keys_.assign(cap, -1);
    vals_.resize(cap);
    mask_ = cap - 1;
  }
  int64_t get(int64_t k) const {
    size_t h = slot(k);
    while (keys_[h] != -1) {
      if (keys_[h] == k) return vals_[h];
      h = (h + 1) & mask_;
    }
    return k;
  }
  void put(int64_t k, int64_t v) {
    size_t h = slot(k);
    while (keys_[h] != -1 && keys_[h] != k) h = (h + 1) & mask_;
    keys_[h] = k;
    vals_[h] = v;
  }

 private:
  size_t slot(int64_t k) const {
    uint64_t z = uint64_t(k) * 0x9E3779B97F4A7C15ull;
    return size_t(z ^ (z >> 29)) & mask_;
  }
  std::vector<int64_t> keys_, vals_;
  size_t mask_;
};

// Generator.choice(n, m, replace=False): numpy uses a partial Fisher-Yates
// over arange(n) when n > 10000 and m > n // 50, else Floyd's algorithm
// followed by a shuffle of the m picks.
inline void rng_choice(Pcg64& g, int64_t n, int64_t m, int64_t* out) {
  if (m <= 0) return;
  if (n > 10000 && m > n / 50) {
    SparseSwap perm(size_t(m) * 2);
    const int64_t stop = (n - m) > 1 ? (n - m) : 1;
    for (int64_t i = n - 1; i >= stop; --i) {
      const int64_t j = int64_t(g.bounded(uint64_t(i)));
      const int64_t at_i = perm.get(i);
      const int64_t at_j = perm.get(j);
      perm.put(j, at_i);
      out[i - (n - m)] = at_j;
    }
    if (n - m == 0) out[0] = perm.get(0);  // position 0 is never a swap source
    return;
  }
  // Floyd: pick an unseen value for each slot (j itself on a repeat), then
  // shuffle the picks.  `seen` maps value -> -1 as a set marker.
  SparseSwap seen(size_t(m) * 2);
  for (int64_t j = n - m; j < n; ++j) {
    int64_t v = int64_t(g.bounded(uint64_t(j)));
    if (seen.get(v) == -1) v = j;
    seen.put(v, -1);
    out[j - (n - m)] = v;
  }
  for (int64_t i = m - 1; i >= 1; --i) {
    const int64_t j = int64_t(g.bounded(uint64_t(i)));
    const int64_t t = out[i];
    out[i] = out[j];
    out[j] = t;
  }
}

// fp64 squared distance rounded like numpy's ((a-b)**2).sum(axis=-1) over a
// length-3 axis: ((dx*dx + dy*dy) + dz*dz), no fused multiply-add.
inline double dist2(const double* a, const double* b) {
  const double dx = a[0] - b[0];
  const double dy = a[1] - b[1];
  const double dz = a[2] - b[2];
  return (dx * dx + dy * dy) + dz * dz;
}

// The LIFO split loop of clustering.py:58-85 over the oversize groups of one
// compatibility class.  `groups` holds the oversize groups in ascending
// original group order, each with ascending member ids; `centers` their
// center ids.  `pos(id)` returns a pointer to the id's xyz.  On return,
// groups[0..q) are the (modified) originals and groups[q..) the split-off
// groups in append order; centers is extended alongside.  Returns the number
// of splits performed.
template <class PosFn>
int64_t split_oversize(Pcg64& g, std::vector<std::vector<int64_t>>& groups,
                       std::vector<int64_t>& centers, int64_t max_size, PosFn pos) {
  std::vector<int64_t> stack;
  for (int64_t c = 0; c < int64_t(groups.size()); ++c)
    if (int64_t(groups[c].size()) > max_size) stack.push_back(c);
  std::vector<int64_t> cand, keep, moved;
  int64_t splits = 0;
  while (!stack.empty()) {
    const int64_t c = stack.back();
    stack.pop_back();
    const std::vector<int64_t>& mem = groups[c];
    if (int64_t(mem.size()) <= max_size) continue;
    const int64_t old_center = centers[c];
    cand.clear();
    for (int64_t x : mem)
      if (x != old_center) cand.push_back(x);
    const std::vector<int64_t>& pool = cand.empty() ? mem : cand;
    const int64_t pick = int64_t(g.bounded(uint64_t(pool.size()) - 1));
    const int64_t new_center = pool[size_t(pick)];
    const double* p0 = pos(old_center);
    const double* p1 = pos(new_center);
    keep.clear();
    moved.clear();
    for (int64_t x : mem) {
      const double* px = pos(x);
      // np.argmin over (old, new): ties stay with the old center
      if (dist2(px, p1) < dist2(px, p0))
        moved.push_back(x);
      else
        keep.push_back(x);
    }
    if (keep.empty() || moved.empty()) {
      const size_t half = mem.size() / 2;
      keep.assign(mem.begin(), mem.begin() + half);
      moved.assign(mem.begin() + half, mem.end());
    }
    ++splits;
    const bool keep_big = int64_t(keep.size()) > max_size;
    const bool moved_big = int64_t(moved.size()) > max_size;
    groups[c] = keep;
    groups.push_back(moved);
    centers.push_back(new_center);
    if (keep_big) stack.push_back(c);
    if (moved_big) stack.push_back(int64_t(groups.size()) - 1);
  }
  return splits;
}

}  // namespace vpg

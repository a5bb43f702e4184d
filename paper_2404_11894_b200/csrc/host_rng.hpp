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
#include <algorithm>
#include <cstring>
#include <memory>
#include <stdexcept>
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

// Open-addressing map of the positions a partial Fisher-Yates has written
// (int32 position -> int32 value, packed in one int64; -1 = empty slot).
class SwapTable {
 public:
  explicit SwapTable(size_t expected) {
    size_t cap = 1024;
    while (cap < expected * 2) cap <<= 1;
    slots_.assign(cap, -1);
    mask_ = cap - 1;
  }
  size_t slot(int64_t k) const { return size_t(uint32_t(k) * 0x9E3779B1u) & mask_; }
  void prefetch(int64_t k) const { __builtin_prefetch(&slots_[slot(k)]); }
  int64_t get(int64_t k) const {  // value at position k (k itself if never written)
    size_t h = slot(k);
    for (;;) {
      const int64_t e = slots_[h];
      if (e == -1) return k;
      if ((e >> 32) == k) return int64_t(int32_t(uint32_t(e)));
      h = (h + 1) & mask_;
    }
  }
  void put(int64_t k, int64_t v) {
    size_t h = slot(k);
    while (slots_[h] != -1 && (slots_[h] >> 32) != k) h = (h + 1) & mask_;
    slots_[h] = (k << 32) | int64_t(uint32_t(v));
  }

 private:
  std::vector<int64_t> slots_;
  size_t mask_;
};

// Generator.choice(n, m, replace=False): numpy uses a partial Fisher-Yates
// over arange(n) when n > 10000 and m > n // 50, else Floyd's algorithm
// followed by a shuffle of the m picks.  The swap targets depend only on the
// random stream, so they are drawn first and the swaps replayed over a
// compact table of written positions (prefetched a few steps ahead).
inline void rng_choice(Pcg64& g, int64_t n, int64_t m, int64_t* out) {
  if (m <= 0) return;
  if (n >= (int64_t(1) << 31)) throw std::length_error("choice population exceeds 2^31");
  if (n > 10000 && m > n / 50) {
    const int64_t stop = (n - m) > 1 ? (n - m) : 1;
    const int64_t steps = n - stop;
    std::vector<int32_t> target(size_t(steps > 0 ? steps : 0));
    for (int64_t k = 0; k < steps; ++k) target[k] = int32_t(g.bounded(uint64_t(n - 1 - k)));
    SwapTable tab{size_t(m)};
    for (int64_t k = 0; k < steps; ++k) {
      if (k + 8 < steps) tab.prefetch(target[k + 8]);
      const int64_t i = n - 1 - k, j = target[k];
      const int64_t at_i = tab.get(i);
      out[i - (n - m)] = tab.get(j);
      tab.put(j, at_i);
    }
    if (n - m == 0) out[0] = tab.get(0);  // position 0 is never a swap source
    return;
  }
  // Floyd: an unseen value per slot (j itself on a repeat), then a shuffle.
  SwapTable seen{size_t(m)};  // value -> marker -2 (as a set)
  for (int64_t j = n - m; j < n; ++j) {
    int64_t v = int64_t(g.bounded(uint64_t(j)));
    if (seen.get(v) == -2) v = j;
    seen.put(v, -2);
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

// A group of the split loop: a contiguous range of the flat member arrays.
struct SplitGroup {
  int64_t begin, size;
  int64_t center;  // member id of the center
};

// The LIFO split loop of clustering.py:58-85 over the oversize groups of one
// compatibility class, on flat arrays.  `ids` holds the members of the
// oversize groups back to back (each group ascending, groups in ascending
// original order); `xyz` their positions (3 doubles per slot, moved with the
// ids).  `groups` describes them; `center_xyz[3k..3k+3)` is the position of
// groups[k].center.  Each split partitions its range in place (stable: kept
// members compacted forward, moved ones appended after them), so every final
// group stays a contiguous ascending range.  The squared distance of each
// member to its current center is cached (a split only evaluates the
// distance to the new center; moved members inherit it) and each group knows
// the slot of its center, so no pass searches for it.  On return
// groups[0..q) are the originals (possibly shrunk) and groups[q..) the
// split-off groups in append order.  Returns the number of splits.
inline int64_t split_oversize(Pcg64& g, int32_t* ids, double* xyz, size_t total,
                              std::vector<SplitGroup>& groups, int64_t max_size,
                              const double* center_xyz, int64_t* visits = nullptr) {
  std::unique_ptr<double[]> d0(new double[total + 1]);
  std::vector<int64_t> cslot(groups.size(), -1);  // slot of each group's center, -1 if absent
  for (size_t k = 0; k < groups.size(); ++k) {
    const SplitGroup& gr = groups[k];
    for (int64_t t = gr.begin; t < gr.begin + gr.size; ++t) {
      d0[t] = dist2(&xyz[t * 3], center_xyz + k * 3);
      if (ids[t] == gr.center && cslot[k] < 0) cslot[k] = t;
    }
  }
  std::vector<int64_t> stack;
  for (int64_t c = 0; c < int64_t(groups.size()); ++c)
    if (groups[c].size > max_size) stack.push_back(c);
  std::vector<int32_t> mid;
  std::vector<double> mxyz, md;
  int64_t splits = 0;
  double* __restrict__ dd0 = d0.get();
  while (!stack.empty()) {
    const int64_t c = stack.back();
    stack.pop_back();
    const SplitGroup gr = groups[c];
    if (gr.size <= max_size) continue;
    const int64_t b = gr.begin, e = gr.begin + gr.size;
    if (visits) *visits += gr.size;
    // candidates = members != old center, in member order (clustering.py:65-67)
    const int64_t at = cslot[c] >= 0 ? cslot[c] - b : -1;
    const int64_t pool = at >= 0 ? gr.size - 1 : gr.size;
    int64_t pick;
    if (pool > 0) {
      pick = int64_t(g.bounded(uint64_t(pool) - 1));
      if (at >= 0 && pick >= at) ++pick;
    } else {
      pick = int64_t(g.bounded(uint64_t(gr.size) - 1));
    }
    const int64_t new_center = ids[b + pick];
    const double pn[3] = {xyz[(b + pick) * 3], xyz[(b + pick) * 3 + 1], xyz[(b + pick) * 3 + 2]};
    // one pass: keep members compacted forward in place, moved ones to the side
    if (int64_t(mid.size()) < gr.size) {
      mid.resize(gr.size);
      md.resize(gr.size);
      mxyz.resize(gr.size * 3);
    }
    int64_t wk = b, wm = 0, keep_center = -1, moved_center = -1;
    const int64_t old_slot = cslot[c], new_slot = b + pick;
    for (int64_t t = b; t < e; ++t) {
      const double v = dist2(&xyz[t * 3], pn);
      if (v < dd0[t]) {  // np.argmin over (old, new): ties stay
        if (t == new_slot) moved_center = wm;
        mid[wm] = ids[t];
        md[wm] = v;
        mxyz[wm * 3] = xyz[t * 3];
        mxyz[wm * 3 + 1] = xyz[t * 3 + 1];
        mxyz[wm * 3 + 2] = xyz[t * 3 + 2];
        ++wm;
      } else {
        if (t == old_slot) keep_center = wk;
        if (wk != t) {
          ids[wk] = ids[t];
          dd0[wk] = dd0[t];
          xyz[wk * 3] = xyz[t * 3];
          xyz[wk * 3 + 1] = xyz[t * 3 + 1];
          xyz[wk * 3 + 2] = xyz[t * 3 + 2];
        }
        ++wk;
      }
    }
    const int64_t kept = wk - b, moved = wm;
    if (kept == 0 || moved == 0) {
      // coincident points: halves (clustering.py:75-78).  Nothing was written
      // back, so the range still holds the group in member order.  The second
      // half takes the new center: its cached distances become d(., new).
      const int64_t half = gr.size / 2;
      for (int64_t t = b + half; t < e; ++t) dd0[t] = dist2(&xyz[t * 3], pn);
      groups[c].size = half;
      cslot[c] = (old_slot >= 0 && old_slot < b + half) ? old_slot : -1;
      groups.push_back(SplitGroup{b + half, gr.size - half, new_center});
      cslot.push_back(new_slot >= b + half ? new_slot : -1);
    } else {
      std::memcpy(ids + wk, mid.data(), sizeof(int32_t) * moved);
      std::memcpy(dd0 + wk, md.data(), sizeof(double) * moved);
      std::memcpy(xyz + wk * 3, mxyz.data(), sizeof(double) * 3 * moved);
      groups[c].size = kept;
      cslot[c] = keep_center;
      groups.push_back(SplitGroup{wk, moved, new_center});
      cslot.push_back(moved_center >= 0 ? wk + moved_center : -1);
    }
    ++splits;
    if (groups[c].size > max_size) stack.push_back(c);
    if (groups.back().size > max_size) stack.push_back(int64_t(groups.size()) - 1);
  }
  return splits;
}

}  // namespace vpg

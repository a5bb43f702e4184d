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
#include <chrono>
#include <functional>
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

// Flat member arrays of the split loop, structure of arrays so the distance
// pass vectorises: id, position and the cached squared distance to the
// member's current center.
struct SplitMembers {
  int32_t* id;
  double *x, *y, *z, *d0;
};

// The LIFO split loop of clustering.py:58-85 over the oversize groups of one
// compatibility class.  `m` holds the members of the oversize groups back to
// back (each group ascending, groups in ascending original order) with d0 =
// squared distance to the group's center; `groups` describes them and
// `cslot[k]` is the slot of groups[k]'s center among its members (-1 if the
// center is not a member).  Each split partitions its range in place
// (stable: kept members compacted forward, moved ones appended after them),
// so every final group stays a contiguous ascending range; a split only
// evaluates the distance to the new center (moved members inherit it as
// their d0).  On return groups[0..q) are the originals (possibly shrunk) and
// groups[q..) the split-off groups in append order.  Returns the number of
// splits.
//
// `masks` (optional) holds, for every original group k in order, cnt_k rows
// of ceil(cnt_k / 64) words: bit m of row p = (member m is strictly closer to
// member p than to the group's center) -- the outcome of the group's FIRST
// split for every possible pick, precomputed on the device.  A first split
// then only draws the pick and partitions; later splits compute as usual.
struct SplitStats {  // diagnostics (VPG_DEBUG_TIMING): count / ns / members per split kind
  int64_t n[3] = {0, 0, 0}, ns[3] = {0, 0, 0}, members[3] = {0, 0, 0};
};

// A first split whose two halves both end at most max_size members: the host
// only draws the pick and books the halves; the members are partitioned on
// the device afterwards (begin, size, offset of the pick's mask row).
struct DeferredSplit {
  int64_t begin, size, row;
};

inline int64_t split_oversize_soa(Pcg64& g, SplitMembers m, std::vector<SplitGroup>& groups,
                                  std::vector<int64_t>& cslot, int64_t max_size,
                                  int64_t* visits = nullptr,
                                  const unsigned long long* masks = nullptr,
                                  SplitStats* stats = nullptr,
                                  const int32_t* first_moved = nullptr,
                                  std::vector<DeferredSplit>* deferred = nullptr,
                                  const std::function<void(int64_t)>* need_bulk = nullptr) {
  const size_t n_orig = groups.size();
  std::vector<int64_t> moff(masks ? n_orig : 0);
  std::vector<uint8_t> fresh(masks ? n_orig : 0, 1);
  for (size_t k = 0, o = 0; k < moff.size(); ++k) {
    moff[k] = int64_t(o);
    o += size_t(groups[k].size) * size_t((groups[k].size + 63) / 64);
  }
  std::vector<int64_t> stack;
  for (int64_t c = 0; c < int64_t(groups.size()); ++c)
    if (groups[c].size > max_size) stack.push_back(c);
  // the original group every group's members came from (positions, distances
  // and mask rows may arrive late: need_bulk(original) before touching them)
  std::vector<int32_t> root(need_bulk ? groups.size() : 0);
  for (size_t c = 0; c < root.size(); ++c) root[c] = int32_t(c);
  std::vector<int32_t> mid;
  std::vector<double> mx, my, mz, md, vbuf;
  std::vector<uint8_t> flag;
  int64_t splits = 0;
  int32_t* __restrict__ id = m.id;
  double* __restrict__ X = m.x;
  double* __restrict__ Y = m.y;
  double* __restrict__ Z = m.z;
  double* __restrict__ D0 = m.d0;
  while (!stack.empty()) {
    const int64_t c = stack.back();
    stack.pop_back();
    const SplitGroup gr = groups[c];
    if (gr.size <= max_size) continue;
    const auto t_start = stats ? std::chrono::steady_clock::now()
                               : std::chrono::steady_clock::time_point();
    auto stat = [&](int kind) {
      if (!stats) return;
      stats->n[kind] += 1;
      stats->members[kind] += gr.size;
      stats->ns[kind] += std::chrono::duration_cast<std::chrono::nanoseconds>(
                             std::chrono::steady_clock::now() - t_start).count();
    };
    const int64_t b = gr.begin, e = gr.begin + gr.size, sz = gr.size;
    if (visits) *visits += sz;
    // candidates = members != old center, in member order (clustering.py:65-67)
    const int64_t at = cslot[c] >= 0 ? cslot[c] - b : -1;
    const int64_t pool = at >= 0 ? sz - 1 : sz;
    int64_t pick;
    if (pool > 0) {
      pick = int64_t(g.bounded(uint64_t(pool) - 1));
      if (at >= 0 && pick >= at) ++pick;
    } else {
      pick = int64_t(g.bounded(uint64_t(sz) - 1));
    }
    const bool first = masks && size_t(c) < n_orig && fresh[c];
    if (first && first_moved) {
      // the staging is fresh from DMA (not in any CPU cache) and originals
      // are popped in descending order: pull a later group's lines in now
      const int64_t ahead = c - 12;
      if (ahead >= 0) {
        const SplitGroup& ga = groups[ahead];
        for (int64_t t = ga.begin; t < ga.begin + ga.size; t += 16) {
          __builtin_prefetch(first_moved + t);
          __builtin_prefetch(id + t);
        }
        // a large group (> 3/2 of the limit) is likely split again: its
        // positions and distances are needed too
        if (2 * ga.size > 3 * max_size)
          for (int64_t t = ga.begin; t < ga.begin + ga.size; t += 8) {
            __builtin_prefetch(X + t);
            __builtin_prefetch(Y + t);
            __builtin_prefetch(Z + t);
            __builtin_prefetch(D0 + t);
          }
      }
    }
    const int64_t new_center = id[b + pick];
    if (first && first_moved && deferred) {
      // first split of an original group, its size known without the row: a
      // final one is booked only (members partitioned on the device)
      const int64_t moved = first_moved[b + pick], kept = sz - moved;
      if (kept > 0 && moved > 0 && kept <= max_size && moved <= max_size) {
        fresh[c] = 0;
        deferred->push_back(DeferredSplit{b, sz, moff[c] + pick * ((sz + 63) / 64)});
        groups[c].size = kept;
        cslot[c] = -1;
        groups.push_back(SplitGroup{b + kept, moved, new_center});
        cslot.push_back(-1);
        if (need_bulk) root.push_back(root[c]);
        ++splits;
        stat(0);
        continue;
      }
    }
    if (need_bulk) (*need_bulk)(root[c]);
    const double px = X[b + pick], py = Y[b + pick], pz = Z[b + pick];
    if (int64_t(mid.size()) < sz) {
      for (auto* v : {&mx, &my, &mz, &md, &vbuf}) v->resize(sz);
      mid.resize(sz);
      flag.resize(sz);
    }
    if (first) {
      // first split of an original group: the moved set is row `pick`
      fresh[c] = 0;
      const int64_t words = (sz + 63) / 64;
      const unsigned long long* row = masks + moff[c] + pick * words;
      int64_t moved = 0;
      for (int64_t w = 0; w < words; ++w) moved += __builtin_popcountll(row[w]);
      const int64_t kept = sz - moved;
      const int64_t old_slot = cslot[c], new_slot = b + pick;
      if (kept > 0 && moved > 0) {
        // stable partition by the row's bits; positions and distances move
        // too only when a half will be split again (its d0 = distance to its
        // center: unchanged for the kept half, to the pick for the moved one)
        // positions only matter for a half that is split again (the other
        // half is final: only its ids are read from here on)
        const bool again_k = kept > max_size, again_m = moved > max_size;
        const bool again = again_k || again_m;
        int32_t* __restrict__ Mi = mid.data();
        double* __restrict__ MX = mx.data();
        double* __restrict__ MY = my.data();
        double* __restrict__ MZ = mz.data();
        double* __restrict__ MD = md.data();
        int64_t wk = b, wm = 0, keep_center = -1, moved_center = -1;
        for (int64_t t = b; t < e; ++t) {
          const int i = int(t - b);
          const int f = int((row[i >> 6] >> (i & 63)) & 1ull);
          const int32_t idv = id[t];
          if (again_k) {
            X[wk] = X[t]; Y[wk] = Y[t]; Z[wk] = Z[t]; D0[wk] = D0[t];
          }
          if (again_m) {
            const double xv = X[t], yv = Y[t], zv = Z[t];
            const double dx = xv - px, dy = yv - py, dz = zv - pz;
            MX[wm] = xv; MY[wm] = yv; MZ[wm] = zv; MD[wm] = (dx * dx + dy * dy) + dz * dz;
          }
          id[wk] = idv;
          Mi[wm] = idv;
          keep_center = (t == old_slot && !f) ? wk : keep_center;
          moved_center = (t == new_slot && f) ? wm : moved_center;
          wk += 1 - f;
          wm += f;
        }
        std::memcpy(id + wk, Mi, sizeof(int32_t) * moved);
        if (again_m) {
          std::memcpy(X + wk, MX, sizeof(double) * moved);
          std::memcpy(Y + wk, MY, sizeof(double) * moved);
          std::memcpy(Z + wk, MZ, sizeof(double) * moved);
          std::memcpy(D0 + wk, MD, sizeof(double) * moved);
        }
        groups[c].size = kept;
        cslot[c] = keep_center;
        groups.push_back(SplitGroup{wk, moved, new_center});
        cslot.push_back(moved_center >= 0 ? wk + moved_center : -1);
        if (need_bulk) root.push_back(root[c]);
        ++splits;
        if (groups[c].size > max_size) stack.push_back(c);
        if (groups.back().size > max_size) stack.push_back(int64_t(groups.size()) - 1);
        stat(again ? 1 : 0);
        continue;
      }
      // coincident points (all or nothing moves): the general path below
      // reproduces the halving with exact distances
    }
    // pass 1 (vectorisable): distance to the new center, np.argmin over
    // (old, new) with ties staying (clustering.py:69-74)
    double* __restrict__ vb = vbuf.data();
    uint8_t* __restrict__ fl = flag.data();
    int64_t moved = 0;
    for (int64_t i = 0; i < sz; ++i) {
      const double dx = X[b + i] - px, dy = Y[b + i] - py, dz = Z[b + i] - pz;
      const double v = (dx * dx + dy * dy) + dz * dz;
      vb[i] = v;
      const uint8_t f = v < D0[b + i];
      fl[i] = f;
      moved += f;
    }
    const int64_t kept = sz - moved;
    const int64_t old_slot = cslot[c], new_slot = b + pick;
    if (kept == 0 || moved == 0) {
      // coincident points: halves (clustering.py:75-78); the range still holds
      // the group in member order.  The second half takes the new center: its
      // cached distances become d(., new).
      const int64_t half = sz / 2;
      for (int64_t t = b + half; t < e; ++t) D0[t] = vb[t - b];
      groups[c].size = half;
      cslot[c] = (old_slot >= 0 && old_slot < b + half) ? old_slot : -1;
      groups.push_back(SplitGroup{b + half, sz - half, new_center});
      cslot.push_back(new_slot >= b + half ? new_slot : -1);
      if (need_bulk) root.push_back(root[c]);
    } else {
      // pass 2: stable partition, branch-free (every slot is written on both
      // sides; a slot is only ever written at or before the one being read)
      int32_t* __restrict__ Mi = mid.data();
      double* __restrict__ MX = mx.data();
      double* __restrict__ MY = my.data();
      double* __restrict__ MZ = mz.data();
      double* __restrict__ MD = md.data();
      int64_t wk = b, wm = 0, keep_center = -1, moved_center = -1;
      for (int64_t t = b; t < e; ++t) {
        const int64_t i = t - b;
        const int32_t f = fl[i];
        const int32_t idv = id[t];
        const double xv = X[t], yv = Y[t], zv = Z[t], d0v = D0[t];
        id[wk] = idv; X[wk] = xv; Y[wk] = yv; Z[wk] = zv; D0[wk] = d0v;
        Mi[wm] = idv; MX[wm] = xv; MY[wm] = yv; MZ[wm] = zv; MD[wm] = vb[i];
        keep_center = (t == old_slot && !f) ? wk : keep_center;
        moved_center = (t == new_slot && f) ? wm : moved_center;
        wk += 1 - f;
        wm += f;
      }
      std::memcpy(id + wk, Mi, sizeof(int32_t) * moved);
      std::memcpy(X + wk, MX, sizeof(double) * moved);
      std::memcpy(Y + wk, MY, sizeof(double) * moved);
      std::memcpy(Z + wk, MZ, sizeof(double) * moved);
      std::memcpy(D0 + wk, MD, sizeof(double) * moved);
      groups[c].size = kept;
      cslot[c] = keep_center;
      groups.push_back(SplitGroup{wk, moved, new_center});
      cslot.push_back(moved_center >= 0 ? wk + moved_center : -1);
      if (need_bulk) root.push_back(root[c]);
    }
    ++splits;
    if (groups[c].size > max_size) stack.push_back(c);
    if (groups.back().size > max_size) stack.push_back(int64_t(groups.size()) - 1);
    stat(2);
  }
  return splits;
}

// AoS entry (tests, vpg_split_groups): positions 3 doubles per slot, the
// centers' positions in center_xyz; d0 and the center slots computed here.
inline int64_t split_oversize(Pcg64& g, int32_t* ids, double* xyz, size_t total,
                              std::vector<SplitGroup>& groups, int64_t max_size,
                              const double* center_xyz, int64_t* visits = nullptr) {
  std::vector<double> x(total + 1), y(total + 1), z(total + 1), d0(total + 1);
  std::vector<int64_t> cslot(groups.size(), -1);
  for (size_t t = 0; t < total; ++t) {
    x[t] = xyz[t * 3];
    y[t] = xyz[t * 3 + 1];
    z[t] = xyz[t * 3 + 2];
  }
  for (size_t k = 0; k < groups.size(); ++k) {
    const SplitGroup& gr = groups[k];
    for (int64_t t = gr.begin; t < gr.begin + gr.size; ++t) {
      d0[t] = dist2(&xyz[t * 3], center_xyz + k * 3);
      if (ids[t] == gr.center && cslot[k] < 0) cslot[k] = t;
    }
  }
  // the first-split rows the device precomputes in the build (same
  // definition), so this entry exercises the same fast path
  std::vector<unsigned long long> masks;
  for (size_t k = 0; k < groups.size(); ++k) {
    const int64_t b = groups[k].begin, cnt = groups[k].size, words = (cnt + 63) / 64;
    for (int64_t p = 0; p < cnt; ++p)
      for (int64_t w = 0; w < words; ++w) {
        unsigned long long bits = 0;
        for (int64_t mm = w * 64; mm < std::min(cnt, w * 64 + 64); ++mm)
          if (dist2(&xyz[(b + mm) * 3], &xyz[(b + p) * 3]) < d0[b + mm]) bits |= 1ull << (mm - w * 64);
        masks.push_back(bits);
      }
  }
  const int64_t n = split_oversize_soa(g, SplitMembers{ids, x.data(), y.data(), z.data(), d0.data()},
                                       groups, cslot, max_size, visits, masks.data());
  for (size_t t = 0; t < total; ++t) {
    xyz[t * 3] = x[t];
    xyz[t * 3 + 1] = y[t];
    xyz[t * 3 + 2] = z[t];
  }
  return n;
}

}  // namespace vpg

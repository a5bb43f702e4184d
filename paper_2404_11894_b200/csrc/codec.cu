// VPGR record blocks <-> device structure-of-arrays (records.py:191-256).
//
// A dump stores records (290 B) and paths (188 B) as packed rows.  Loading
// one on the device is a single host->device copy of the packed block and
// this transposition; saving from the device is the reverse.  A warp stages
// 32 consecutive rows in shared memory with coalesced 16-byte loads, then
// each lane moves its row's fields (unaligned inside the row) into the
// per-field arrays, so both sides of the copy stay coalesced.
#include <cstring>

#include "internal.cuh"

namespace vpg {
namespace {

constexpr int kCodecWarps = 4;
constexpr int kMaxRowBytes = 304;  // >= the widest packed row (290 B records)

struct FieldTable {
  int32_t n;
  int32_t offset[VPG_CODEC_MAX_FIELDS];
  int32_t bytes[VPG_CODEC_MAX_FIELDS];
  uint8_t* ptr[VPG_CODEC_MAX_FIELDS];
};

template <bool kUnpack>
__global__ void __launch_bounds__(kCodecWarps * 32)
k_codec(uint8_t* __restrict__ packed, int64_t n, int row_bytes, FieldTable ft) {
  __shared__ __align__(16) uint8_t stage[kCodecWarps][32 * kMaxRowBytes];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint8_t* st = stage[wid];
  const int64_t step = int64_t(gridDim.x) * kCodecWarps * 32;
  for (int64_t base = (int64_t(blockIdx.x) * kCodecWarps + wid) * 32; base < n; base += step) {
    const int rows = int(n - base < 32 ? n - base : 32);
    const int64_t nbytes = int64_t(rows) * row_bytes;
    uint8_t* blk = packed + base * row_bytes;
    if (kUnpack) {
      // the block is contiguous; 16-byte words when aligned, else bytes
      if ((reinterpret_cast<uintptr_t>(blk) & 15) == 0 && nbytes % 16 == 0) {
        for (int64_t w = lane; w < nbytes / 16; w += 32)
          reinterpret_cast<uint4*>(st)[w] = reinterpret_cast<const uint4*>(blk)[w];
      } else {
        for (int64_t b = lane; b < nbytes; b += 32) st[b] = blk[b];
      }
      __syncwarp();
      if (lane < rows)
        for (int f = 0; f < ft.n; ++f)
          memcpy(ft.ptr[f] + (base + lane) * ft.bytes[f], st + lane * row_bytes + ft.offset[f],
                 size_t(ft.bytes[f]));
    } else {
      if (lane < rows)
        for (int f = 0; f < ft.n; ++f)
          memcpy(st + lane * row_bytes + ft.offset[f], ft.ptr[f] + (base + lane) * ft.bytes[f],
                 size_t(ft.bytes[f]));
      __syncwarp();
      if ((reinterpret_cast<uintptr_t>(blk) & 15) == 0 && nbytes % 16 == 0) {
        for (int64_t w = lane; w < nbytes / 16; w += 32)
          reinterpret_cast<uint4*>(blk)[w] = reinterpret_cast<const uint4*>(st)[w];
      } else {
        for (int64_t b = lane; b < nbytes; b += 32) blk[b] = st[b];
      }
    }
    __syncwarp();
  }
}

}  // namespace

void codec_rows(bool unpack, uint8_t* packed, int64_t n, int32_t row_bytes,
                const vpg_codec_field* fields, int32_t n_fields, cudaStream_t s) {
  VPG_REQUIRE(n_fields >= 0 && n_fields <= VPG_CODEC_MAX_FIELDS, VPG_ELIMIT, "too many fields");
  VPG_REQUIRE(row_bytes > 0 && row_bytes <= kMaxRowBytes, VPG_ELIMIT, "packed row too wide");
  FieldTable ft{};
  ft.n = n_fields;
  for (int f = 0; f < n_fields; ++f) {
    VPG_REQUIRE(fields[f].offset >= 0 && fields[f].bytes > 0 &&
                    fields[f].offset + fields[f].bytes <= row_bytes,
                VPG_EINVAL, "field outside the packed row");
    ft.offset[f] = fields[f].offset;
    ft.bytes[f] = fields[f].bytes;
    ft.ptr[f] = static_cast<uint8_t*>(fields[f].ptr);
  }
  if (n <= 0) return;
  const int64_t warps = (n + 31) / 32;
  const int grid = int(std::min<int64_t>((warps + kCodecWarps - 1) / kCodecWarps, sm_count() * 8));
  if (unpack)
    VPG_LAUNCH(k_codec<true>, grid, kCodecWarps * 32, 0, s, packed, n, row_bytes, ft);
  else
    VPG_LAUNCH(k_codec<false>, grid, kCodecWarps * 32, 0, s, packed, n, row_bytes, ft);
}

}  // namespace vpg

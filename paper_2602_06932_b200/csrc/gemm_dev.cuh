// gemm_dev.cuh — device helpers shared by the tcgen05 GEMM engine (k_gemm.cu) and the
// fused persistent backward kernel (k_bwd.cu).
#pragma once
#include <cfloat>
#include <climits>

#include "internal.h"
#include "ptx.cuh"

namespace aur {
constexpr float kLog2e = 1.4426950408889634f;

template <bool MN>
__device__ __forceinline__ uint64_t operand_desc(uint32_t tile_base, int k) {
  // K-major SW128: rows of 128 B (64 bf16 of K), 8-row atoms 1024 B apart (SBO);
  //   advancing K by 16 elements moves the start address by 32 B inside the atom.
  // MN-major SW128: 64-element MN slices of [BK rows x 128 B] (8 KB, LBO) ;
  //   8-row K groups 1024 B apart (SBO); advancing K by 16 rows = 2048 B.
  if constexpr (MN) {
    return umma_desc_sw128(tile_base + static_cast<uint32_t>(k) * 2048u, BK * 128u, 1024u);
  } else {
    return umma_desc_sw128(tile_base + static_cast<uint32_t>(k) * 32u, 16u, 1024u);
  }
}

__device__ __forceinline__ float select32(const float (&z)[32], int j) {
  float v = 0.f;
#pragma unroll
  for (int jj = 0; jj < 32; ++jj) v = (jj == j) ? z[jj] : v;
  return v;
}

// Tile raster: m-fastest (default: consecutive units share the B tile, so the large B
// operand streams once) or n-fastest (the large operand is A, e.g. dZ^T in the dW GEMM).
__device__ __forceinline__ void decode_unit(const GemmArgs& a, int u, int& mt, int& nt, int& sp) {
  if (a.group > 0) {
    // grouped raster (large operands on both sides, F4 projections): units sweep the other
    // dimension inside groups of `group` tiles, so the group's blocks stay in L2 while the
    // other operand's block is reused `group` times
    const int per = a.m_tiles * a.n_tiles;
    sp = u / per;
    const int v = u - sp * per;
    const int outer = a.group_on_n ? a.n_tiles : a.m_tiles, inner_n = a.group_on_n ? a.m_tiles : a.n_tiles;
    const int g = v / (a.group * inner_n);
    const int first = g * a.group;
    const int gs = min(a.group, outer - first);
    const int w = v - g * a.group * inner_n;
    const int in_grp = first + w % gs, other = w / gs;
    if (a.group_on_n) { nt = in_grp; mt = other; }
    else { mt = in_grp; nt = other; }
    return;
  }
  if (a.n_fastest) {
    nt = u % a.n_tiles;
    const int rest = u / a.n_tiles;
    mt = rest % a.m_tiles;
    sp = rest / a.m_tiles;
  } else {
    mt = u % a.m_tiles;
    const int rest = u / a.m_tiles;
    nt = rest % a.n_tiles;
    sp = rest / a.n_tiles;
  }
}

struct SupCursor {
  const int32_t* idx;
  const float* p;
  int k;
  int pos;
  int64_t nxt;  // local GEMM column of the next support entry (INT64_MAX = none)
  float nxt_p;
  int64_t limit;  // valid columns (entries at/after limit are ignored)
  int64_t gid0;
  __device__ __forceinline__ void load() {
    nxt = INT64_MAX;
    nxt_p = 0.f;
    while (pos < k) {
      const int32_t g = idx[pos];
      if (g == INT32_MAX) { pos = k; break; }
      const int64_t loc = static_cast<int64_t>(g) - gid0;
      if (loc >= limit) { pos = k; break; }
      nxt = loc;
      nxt_p = p[pos];
      return;
    }
  }
  // position on the first entry with local column >= col0: lower_bound over the
  // index-sorted support (INT32_MAX padding sorts last); O(log k) for supports up to 1024
  __device__ __forceinline__ void seek(int64_t col0) {
    const int64_t target = gid0 + col0;
    int lo = 0, hi = k;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (static_cast<int64_t>(idx[mid]) < target) lo = mid + 1;
      else hi = mid;
    }
    pos = lo;
    load();
  }
  __device__ __forceinline__ void advance() {
    ++pos;
    load();
  }
};

// Runtime-major operand descriptor (fused bwd: the major-ness varies per tile type).
__device__ __forceinline__ uint64_t operand_desc_rt(uint32_t tile_base, int k, bool mn) {
  return mn ? umma_desc_sw128(tile_base + static_cast<uint32_t>(k) * 2048u, BK * 128u, 1024u)
            : umma_desc_sw128(tile_base + static_cast<uint32_t>(k) * 32u, 16u, 1024u);
}

}  // namespace aur

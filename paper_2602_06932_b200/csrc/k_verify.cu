// k_verify.cu — greedy verification / label extraction.
//
//   k_target_scan   A2  one pass over the verifier logits (HBM-bound): per (row, vocab
//                       segment) top-k_max by (value desc, index asc), exact bf16 compares
//                       (P:120 greedy argmax; ties S:84/S:207).  16-byte loads, 8 in flight.
//   k_topk_merge    A2  merges the segment lists of a row (warp per row) -> y_m, top list.
//   k_verify        A3  warp per request, lane = node: match, pointer-jumping ancestor AND,
//                       lowest-index sibling wins; accept_len, bonus, row classes (P:120,
//                       P:179).
//   k_finalize      A4  supports, p~ = renormalised target softmax, H~, weights (Eq. 3,
//                       P:188-195).
#include <cfloat>
#include <climits>

#include "internal.h"
#include "ptx.cuh"

namespace aur {

namespace {
constexpr int KM = AURORA_MAX_K;  // maximum list length (runtime k <= KM <= 32 lanes)

// (v, i) ranks before (w, j)?  value desc, index asc (numeric compare: -0 == +0).
__device__ __forceinline__ bool better(float v, int32_t i, float w, int32_t j) {
  return v > w || (v == w && i < j);
}

// A sorted top-k list distributed over the lanes of a warp: lane j holds entry j
// ((value desc, index asc)); lanes >= k hold spilled / sentinel entries.  All lanes
// call every member with warp-uniform arguments.
struct WarpList {
  float v;
  int32_t i;
  float thr_v;    // entry k-1 (the admission threshold)
  int32_t thr_i;
  int k;
  __device__ __forceinline__ void init(int k_) {
    v = -INFINITY; i = INT32_MAX; thr_v = -INFINITY; thr_i = INT32_MAX; k = k_;
  }
  __device__ __forceinline__ bool admits(float cv, int32_t ci) const { return better(cv, ci, thr_v, thr_i); }
  // insert a warp-uniform candidate that admits() accepted
  __device__ __forceinline__ void insert(float cv, int32_t ci) {
    const int lane = threadIdx.x & 31;
    const uint32_t b = __ballot_sync(0xffffffffu, better(cv, ci, v, i));
    const int pos = __ffs(b) - 1;  // >= 0 because the candidate beats entry k-1
    const float uv = __shfl_up_sync(0xffffffffu, v, 1);
    const int32_t ui = __shfl_up_sync(0xffffffffu, i, 1);
    if (lane > pos) { v = uv; i = ui; }
    if (lane == pos) { v = cv; i = ci; }
    thr_v = __shfl_sync(0xffffffffu, v, k - 1);
    thr_i = __shfl_sync(0xffffffffu, i, k - 1);
  }
  // offer one value held by lane `src` (warp-uniform src)
  __device__ __forceinline__ void offer(float myv, int32_t myi, int src) {
    const float cv = __shfl_sync(0xffffffffu, myv, src);
    const int32_t ci = __shfl_sync(0xffffffffu, myi, src);
    if (admits(cv, ci)) insert(cv, ci);
  }
};

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pick4(const uint4& w, int e) {
  return e == 0 ? w.x : (e == 1 ? w.y : (e == 2 ? w.z : w.w));
}
__device__ __forceinline__ uint32_t nonfinite8(const uint4& w) {
  const uint32_t ax = __vmaxu2(__vmaxu2(w.x & 0x7FFF7FFFu, w.y & 0x7FFF7FFFu),
                               __vmaxu2(w.z & 0x7FFF7FFFu, w.w & 0x7FFF7FFFu));
  return static_cast<uint32_t>((ax & 0xFFFFu) >= 0x7F80u) | static_cast<uint32_t>((ax >> 16) >= 0x7F80u);
}
__device__ __forceinline__ float max8(const uint4& w) {
  const __nv_bfloat162 m2 = __hmax2(__hmax2(*reinterpret_cast<const __nv_bfloat162*>(&w.x),
                                            *reinterpret_cast<const __nv_bfloat162*>(&w.y)),
                                    __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&w.z),
                                            *reinterpret_cast<const __nv_bfloat162*>(&w.w)));
  return fmaxf(__low2float(m2), __high2float(m2));
}
// Order-preserving float <-> int map (signed-int order == float order) for smem atomicMax.
__device__ __forceinline__ int f2ord(float f) { const int i = __float_as_int(f); return i >= 0 ? i : i ^ 0x7FFFFFFF; }
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }
__device__ __forceinline__ float elem8(const uint4& w, int e) {
  const uint32_t word = pick4(w, e >> 1);
  return (e & 1) ? bf16_hi(word) : bf16_lo(word);
}
// Each lane holds one 8-element vector starting at column `col`.  Elements >= floor
// are offered one by one (warp-uniform order); the exact (value, index) admission test
// against the list's k-th entry happens at insertion.
__device__ __forceinline__ void offer_vectors(WarpList& L, bool lane_hit, const uint4& w, int64_t col, float floor) {
  uint32_t my = 0;
  if (lane_hit) {
#pragma unroll
    for (int e = 0; e < 8; ++e) my |= (elem8(w, e) >= fmaxf(floor, L.thr_v) ? 1u : 0u) << e;
  }
  uint32_t lanes = __ballot_sync(0xffffffffu, my != 0);
  while (lanes) {
    const int src = __ffs(lanes) - 1;
    const int e = __shfl_sync(0xffffffffu, __ffs(my) - 1, src);
    const float cv = __shfl_sync(0xffffffffu, elem8(w, e), src);
    const int32_t ci = static_cast<int32_t>(__shfl_sync(0xffffffffu, col, src) + e);
    if (threadIdx.x % 32 == static_cast<unsigned>(src)) my &= my - 1;
    if (cv >= floor && L.admits(cv, ci)) L.insert(cv, ci);
    lanes = __ballot_sync(0xffffffffu, my != 0);
  }
}
// k-th largest of the 32 lane values (k <= 32): a valid lower bound for the k-th best
// element when every lane value is itself an element.
__device__ __forceinline__ float warp_kth_largest(float x, int k) {
  float kth = -INFINITY;
  for (int r = 0; r < k; ++r) {
    float m = x;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    kth = m;
    const uint32_t eq = __ballot_sync(0xffffffffu, x == m);
    if ((threadIdx.x & 31) == static_cast<unsigned>(__ffs(eq) - 1)) x = -INFINITY;
  }
  return kth;
}
__device__ __forceinline__ uint4 ld_nc_v4(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
}  // namespace

// --------------------------------------------------------------------------- A2 scan
// grid (M * nseg), 256 threads = 8 warps.  Segment [seg*seg_len, min(V_local, +seg_len)).
// Each warp keeps a lane-distributed top-k; a lane's 8 bf16 (one 16 B load) are only
// offered when their bf16x2 max reaches the warp's k-th value, so after warm-up almost
// every 16 B costs a handful of instructions (HBM-bound).
__global__ void __launch_bounds__(256) k_target_scan(VerifyLaunch p) {
  const int row = blockIdx.x / p.nseg;
  const int seg = blockIdx.x % p.nseg;
  const int k = p.k_max;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c0 = static_cast<int64_t>(seg) * p.seg_len;
  const int64_t c1 = min(p.V_local, c0 + p.seg_len);
  const uint16_t* T = p.T + static_cast<int64_t>(row) * p.ldT;
  WarpList L;
  L.init(k);
  uint32_t bad = 0;
  __shared__ int s_floor;  // max over warps of their k-th value: a CTA-wide admission floor
  if (threadIdx.x == 0) s_floor = f2ord(-INFINITY);
  __syncthreads();
  float floor = -INFINITY;

  const bool aligned = ((reinterpret_cast<uintptr_t>(T + c0) & 15) == 0);
  const int64_t nvec = aligned ? (c1 - c0) >> 3 : 0;
  const uint4* src = reinterpret_cast<const uint4*>(T + c0);
  constexpr int U = 8;  // 16 B loads in flight per lane
  // vectors are interleaved: warp w handles [w*32 + i*256, +32) for i = 0, 1, ...
  int64_t base = static_cast<int64_t>(warp) * 32;
  {
    // ---- CTA-wide warm start: every warp loads its first batch, the 256 lane maxima
    // (distinct elements) go to smem, and the k-th largest of them is a valid lower
    // bound for the k-th best element of the segment.
    __shared__ float s_lm[256];
    uint4 w[U];
    float gm[U];
    float lm = -INFINITY;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t vi = base + u * 256 + lane;
      w[u] = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
      if (vi < nvec) {
        w[u] = ld_nc_v4(src + vi);
        bad |= nonfinite8(w[u]);
      }
      gm[u] = max8(w[u]);
      lm = fmaxf(lm, gm[u]);
    }
    s_lm[threadIdx.x] = lm;
    __syncthreads();
    float v8[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v8[j] = s_lm[lane * 8 + j];
    for (int r = 0; r < k; ++r) {
      float m = v8[0];
#pragma unroll
      for (int j = 1; j < 8; ++j) m = fmaxf(m, v8[j]);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
      if (r == k - 1) floor = fmaxf(floor, m);
      const uint32_t has = __ballot_sync(0xffffffffu, v8[0] == m || v8[1] == m || v8[2] == m || v8[3] == m ||
                                                          v8[4] == m || v8[5] == m || v8[6] == m || v8[7] == m);
      if (lane == __ffs(has) - 1) {
        bool done = false;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const bool hit = !done && v8[j] == m;
          v8[j] = hit ? -INFINITY : v8[j];
          done = done || hit;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t vi = base + u * 256 + lane;
      const bool h = vi < nvec && gm[u] >= fmaxf(floor, L.thr_v);
      if (__any_sync(0xffffffffu, h)) offer_vectors(L, h, w[u], c0 + vi * 8, floor);
    }
    base += U * 256;
  }
  for (; base + (U - 1) * 256 + 31 < nvec; base += U * 256) {
    uint4 w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) w[u] = ld_nc_v4(src + base + u * 256 + lane);
    float gm[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      bad |= nonfinite8(w[u]);
      gm[u] = max8(w[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool h = gm[u] >= fmaxf(floor, L.thr_v);
      if (__any_sync(0xffffffffu, h)) offer_vectors(L, h, w[u], c0 + (base + u * 256 + lane) * 8, floor);
    }
    // share this warp's k-th value with the CTA; pick up the others'
    if (lane == 0 && L.thr_v > floor) atomicMax(&s_floor, f2ord(L.thr_v));
    floor = fmaxf(floor, ord2f(*reinterpret_cast<volatile int*>(&s_floor)));
  }
  for (; base < nvec; base += 256) {
    const int64_t vi = base + lane;
    uint4 w = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);  // -inf padding
    if (vi < nvec) {
      w = ld_nc_v4(src + vi);
      bad |= nonfinite8(w);
    }
    const float gm = max8(w);
    const bool h = vi < nvec && gm >= fmaxf(floor, L.thr_v);
    if (__any_sync(0xffffffffu, h)) offer_vectors(L, h, w, c0 + vi * 8, floor);
  }
  // scalar tail (or whole segment when the row start is not 16 B aligned)
  for (int64_t cb = c0 + nvec * 8 + static_cast<int64_t>(warp) * 32; cb < c1; cb += 256) {
    const int64_t col = cb + lane;
    float v = -INFINITY;
    if (col < c1) {
      const uint32_t b = T[col];
      bad |= static_cast<uint32_t>((b & 0x7FFFu) >= 0x7F80u);
      v = __uint_as_float(b << 16);
    }
    uint32_t hit = __ballot_sync(0xffffffffu, col < c1 && v >= floor && L.admits(v, static_cast<int32_t>(col)));
    while (hit) {
      const int s = __ffs(hit) - 1;
      hit &= hit - 1;
      L.offer(v, static_cast<int32_t>(col), s);
    }
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (bad && lane == 0) atomicOr(p.lab.status, AURORA_STATUS_NONFINITE);

  // ---- block merge: warp lists -> smem -> warp 0
  __shared__ float s_v[8][KM];
  __shared__ int32_t s_i[8][KM];
  if (lane < k) { s_v[warp][lane] = L.v; s_i[warp][lane] = L.i; }
  __syncthreads();
  if (warp == 0) {
    WarpList F;
    F.init(k);
    for (int w8 = 0; w8 < 8; ++w8) {
      const float cv = lane < k ? s_v[w8][lane] : -INFINITY;
      const int32_t ci = lane < k ? s_i[w8][lane] : INT32_MAX;
      uint32_t hit = __ballot_sync(0xffffffffu, lane < k && F.admits(cv, ci));
      while (hit) {
        const int s = __ffs(hit) - 1;
        hit &= hit - 1;
        F.offer(cv, ci, s);
      }
    }
    if (lane < k) {
      const int64_t o = (static_cast<int64_t>(row) * p.nseg + seg) * k;
      p.cand_val[o + lane] = F.v;
      p.cand_idx[o + lane] = (F.i == INT32_MAX) ? INT32_MAX : static_cast<int32_t>(F.i + p.vocab_offset);
    }
  }
}

// --------------------------------------------------------------------------- A2 scan (flat split)
// Persistent, load-balanced variant (rows 16 B aligned, V_local % 8 == 0): the M x V_local/8
// 16-byte vectors of the batch, flattened row-major, are cut into W equal contiguous ranges, one
// per warp of a grid of `ctas_per_sm` x 148 CTAs, so every warp streams the same number of bytes
// and no wave tail is left (the (row, segment) grid leaves one: M = 1792 rows over 444 resident
// CTAs is 4.04 waves).  A range covers pieces of one or more rows; each piece gets its own list
// (warm start: the k-th largest lane maximum of its first batch) written to slot
// (warp - first warp of the row) of the row's S list slots; the warp that ends a row fills the
// row's remaining slots with empty lists, so the merge reads exactly S lists per row.
struct FlatSplit {
  int64_t V8, NV;  // vectors per row, vectors in the batch
  int32_t W, S;    // warps with a range (each >= 64 vectors), list slots per row
  __device__ __host__ __forceinline__ int64_t start(int64_t g) const { return g * NV / W; }
  // the warp whose range contains vector v: largest g with start(g) <= v
  __device__ __forceinline__ int64_t warp_of(int64_t v) const {
    int64_t g = ((v + 1) * W + NV - 1) / NV - 1;
    while (g + 1 < W && start(g + 1) <= v) ++g;
    while (g > 0 && start(g) > v) --g;
    return g;
  }
};

// Scan vectors [v0, v1) of one row (rowv: the row's first vector) into the warp list L.
// `slot` (shared memory, may be null) is the row's CTA-wide admission floor: every warp of the CTA
// scanning a piece of the same row publishes its k-th value there and admits only elements >= the
// maximum published (a lower bound for the row's k-th best), so the warps' lists stay short.
// Returns this lane's running maximum of |bits| (non-finite test at the end).
__device__ __forceinline__ uint32_t scan_piece(WarpList& L, const uint4* __restrict__ rowv, int64_t v0, int64_t v1,
                                               int* slot, uint4* stash, float f0, bool own_warm) {
  constexpr int U = 8;  // 16 B loads per lane per batch (two batches in flight)
  const int lane = threadIdx.x & 31;
  uint32_t amax = 0;
  auto absmax = [&](const uint4& w) {
    amax = __vmaxu2(amax, __vmaxu2(__vmaxu2(w.x & 0x7FFF7FFFu, w.y & 0x7FFF7FFFu),
                                   __vmaxu2(w.z & 0x7FFF7FFFu, w.w & 0x7FFF7FFFu)));
  };
  float floor = f0;
  {
    // warm start without offers (unless the caller has a floor): the k-th largest of the 32 lane
    // maxima of the first batch (distinct elements) bounds the piece's k-th best element from
    // below; the batch itself is scanned again (from L2) by the main loop
    if (own_warm) {
      float lm = -INFINITY;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t vi = v0 + u * 32 + lane;
        if (vi < v1) lm = fmaxf(lm, max8(ld_nc_v4(rowv + vi)));
      }
      floor = fmaxf(floor, warp_kth_largest(lm, L.k));
    }
    if (slot) {
      if (lane == 0) atomicMax(slot, f2ord(floor));
      floor = fmaxf(floor, ord2f(*reinterpret_cast<volatile int*>(slot)));
    }
  }
  int64_t base = v0;
  // full batches, software-pipelined: the next batch's loads are issued before this one is
  // scanned (two batches in flight per warp while it works), the registers handed over at the end
  uint4 w[U], nx[U];
  if (base + U * 32 <= v1) {
#pragma unroll
    for (int u = 0; u < U; ++u) w[u] = ld_nc_v4(rowv + base + u * 32 + lane);
  }
  for (; base + U * 32 <= v1; base += U * 32) {
    const bool more = base + 2 * U * 32 <= v1;
    if (more) {
#pragma unroll
      for (int u = 0; u < U; ++u) nx[u] = ld_nc_v4(rowv + base + U * 32 + u * 32 + lane);
    }
    uint32_t hm = 0;  // this lane's vectors whose max reaches the admission threshold
    const float f = fmaxf(floor, L.thr_v);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      absmax(w[u]);
      hm |= (max8(w[u]) >= f ? 1u : 0u) << u;
    }
    const uint32_t wm = __reduce_or_sync(0xffffffffu, hm);
    if (wm) {
      // rare path, kept rolled (one copy of the offer code): the batch goes through this warp's
      // shared-memory stash so the hit vectors can be indexed at run time
#pragma unroll
      for (int u = 0; u < U; ++u) stash[u * 32 + lane] = w[u];
      __syncwarp();
#pragma unroll 1
      for (uint32_t mm = wm; mm; mm &= mm - 1) {
        const int u = __ffs(mm) - 1;
        const uint4 wu = stash[u * 32 + lane];
        const bool h = max8(wu) >= fmaxf(floor, L.thr_v);
        if (__any_sync(0xffffffffu, h)) offer_vectors(L, h, wu, (base + u * 32 + lane) * 8, floor);
      }
      __syncwarp();
      if (slot) {
        if (lane == 0 && L.thr_v > floor) atomicMax(slot, f2ord(L.thr_v));
        floor = fmaxf(floor, ord2f(*reinterpret_cast<volatile int*>(slot)));
      }
    } else if (slot) {
      floor = fmaxf(floor, ord2f(*reinterpret_cast<volatile int*>(slot)));
    }
    if (more) {
#pragma unroll
      for (int u = 0; u < U; ++u) w[u] = nx[u];
    }
  }
  for (; base < v1; base += 32) {
    const int64_t vi = base + lane;
    uint4 w = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
    if (vi < v1) {
      w = ld_nc_v4(rowv + vi);
      absmax(w);
    }
    const bool h = vi < v1 && max8(w) >= fmaxf(floor, L.thr_v);
    if (__any_sync(0xffffffffu, h)) offer_vectors(L, h, w, vi * 8, floor);
  }
  return amax;
}

template <int kCtas>
__global__ void __launch_bounds__(256, kCtas) k_target_scan_flat(VerifyLaunch p, FlatSplit fs) {
  constexpr int kSlots = 16;  // rows of the CTA's vector span with a shared admission floor
  __shared__ int s_floor[kSlots];
  __shared__ uint4 s_stash[8][8 * 32];  // per warp: one batch (8 vectors per lane)
  const int lane = threadIdx.x & 31;
  const int64_t g0 = static_cast<int64_t>(blockIdx.x) * 8;
  const int64_t row0 = fs.start(g0 < fs.W ? g0 : fs.W - 1) / fs.V8;
  __shared__ float s_lm[8][32];
  __shared__ int64_t s_row[8];
  if (threadIdx.x < kSlots) s_floor[threadIdx.x] = f2ord(-INFINITY);
  const int warp = threadIdx.x >> 5;
  const int64_t g = g0 + warp;
  const int k = p.k_max;
  int64_t a = g < fs.W ? fs.start(g) : 0;
  const int64_t b = g < fs.W ? fs.start(g + 1) : 0;
  // CTA-wide warm start of every warp's first piece: the 32 lane maxima of each warp's first batch
  // go to shared memory; each warp takes the k-th largest of those of the warps on its row (256
  // distinct elements of the row at most): a much tighter first floor than one warp's 32
  float f0 = -INFINITY;
  {
    constexpr int U = 8;
    float lm = -INFINITY;
    int64_t row = -1;
    if (a < b) {
      row = a / fs.V8;
      const int64_t rs = row * fs.V8, re = min(b, rs + fs.V8);
      const uint4* rowv = reinterpret_cast<const uint4*>(p.T + row * p.ldT);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t vi = a - rs + u * 32 + lane;
        if (vi < re - rs) lm = fmaxf(lm, max8(ld_nc_v4(rowv + vi)));
      }
    }
    s_lm[warp][lane] = lm;
    if (lane == 0) s_row[warp] = row;
    __syncthreads();
    if (row >= 0) {
      float v8[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v8[j] = s_row[j] == row ? s_lm[j][lane] : -INFINITY;
      for (int r = 0; r < k; ++r) {
        float m = v8[0];
#pragma unroll
        for (int j = 1; j < 8; ++j) m = fmaxf(m, v8[j]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
        if (r == k - 1) f0 = m;
        const uint32_t has = __ballot_sync(0xffffffffu, v8[0] == m || v8[1] == m || v8[2] == m || v8[3] == m ||
                                                            v8[4] == m || v8[5] == m || v8[6] == m || v8[7] == m);
        if (lane == __ffs(has) - 1) {
          bool done = false;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const bool hit = !done && v8[j] == m;
            v8[j] = hit ? -INFINITY : v8[j];
            done = done || hit;
          }
        }
      }
    }
  }
  if (g >= fs.W) return;
  uint32_t amax = 0;
  bool first = true;
  while (a < b) {
    const int64_t row = a / fs.V8;
    const int64_t rs = row * fs.V8;
    const int64_t re = min(b, rs + fs.V8);
    WarpList L;
    L.init(k);
    const uint4* rowv = reinterpret_cast<const uint4*>(p.T + row * p.ldT);
    int* slot = row - row0 < kSlots ? &s_floor[row - row0] : nullptr;
    amax = __vmaxu2(amax, scan_piece(L, rowv, a - rs, re - rs, slot, s_stash[warp], first ? f0 : -INFINITY, !first));
    first = false;
    const int64_t sl0 = g - fs.warp_of(rs);
    float* cv = p.cand_val + row * fs.S * k;
    int32_t* ci = p.cand_idx + row * fs.S * k;
    if (lane < k) {
      cv[sl0 * k + lane] = L.v;
      ci[sl0 * k + lane] = (L.i == INT32_MAX) ? INT32_MAX : static_cast<int32_t>(L.i + p.vocab_offset);
    }
    if (re == rs + fs.V8) {  // this warp ends the row: empty lists in the row's unused slots
      for (int64_t sl = sl0 + 1; sl < fs.S; ++sl)
        if (lane < k) { cv[sl * k + lane] = -INFINITY; ci[sl * k + lane] = INT32_MAX; }
    }
    a = re;
  }
  amax = __reduce_max_sync(0xffffffffu, amax);
  if (lane == 0 && ((amax & 0xFFFFu) >= 0x7F80u || (amax >> 16) >= 0x7F80u))
    atomicOr(p.lab.status, AURORA_STATUS_NONFINITE);
}

// --------------------------------------------------------------------------- A2 scan (TMA rings)
// Persistent variant for 16 B-aligned rows.  Every warp owns a private 3-slot ring of 8 KB in
// shared memory and streams its own (row, segment) work items through it: lane 0 issues the 1-D
// bulk async copy (cp.async.bulk) of chunk c + 2 before the warp scans chunk c, so each warp keeps
// 16 KB in flight (128 KB per SM) independently of registers and occupancy, and each item has
// ONE list (the cost of keeping a top-k list is ~k ln(n / k) offers per list: one list per
// 16K+ columns keeps it well below the streaming work).  Warm start per item: the k-th largest
// lane maximum of the first batch bounds the k-th best element from below.
constexpr int kRingChunk = 8192;   // bytes per slot (4096 columns)
constexpr int kRingSlots = 3;
constexpr int kRingWarps = 8;
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__global__ void __launch_bounds__(32 * kRingWarps, 1) k_target_scan_ring(VerifyLaunch p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = base + warp * (kRingSlots * kRingChunk);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + kRingWarps * kRingSlots * kRingChunk) + warp * kRingSlots;
  const int k = p.k_max;
  const int items = p.M * p.nseg;
  if (lane == 0) {
    for (int i = 0; i < kRingSlots; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncwarp();
  uint32_t bad = 0, used = 0;  // chunks consumed by this warp (slot = used % 3, parity = (used / 3) & 1)
  for (int u = blockIdx.x * kRingWarps + warp; u < items; u += gridDim.x * kRingWarps) {
    const int row = u / p.nseg, seg = u % p.nseg;
    const int64_t c0 = static_cast<int64_t>(seg) * p.seg_len;
    const int64_t c1 = min(p.V_local, c0 + p.seg_len);
    const int64_t nvec = c1 > c0 ? (c1 - c0) >> 3 : 0;
    const int64_t vbytes = nvec * 16;
    const int nch = static_cast<int>((vbytes + kRingChunk - 1) / kRingChunk);
    const uint8_t* src = reinterpret_cast<const uint8_t*>(p.T + static_cast<int64_t>(row) * p.ldT + c0);
    auto issue = [&](int c) {  // lane 0: chunk c of this item into slot (used + c) % 3
      const uint32_t slot = (used + c) % kRingSlots;
      const uint32_t bytes = static_cast<uint32_t>(min(static_cast<int64_t>(kRingChunk), vbytes - static_cast<int64_t>(c) * kRingChunk));
      mbar_arrive_expect_tx(&full[slot], bytes);
      bulk_g2s(ring + slot * kRingChunk, src + static_cast<int64_t>(c) * kRingChunk, bytes, &full[slot]);
    };
    if (lane == 0)
      for (int c = 0; c < 2 && c < nch; ++c) issue(c);
    WarpList L;
    L.init(k);
    float floor = -INFINITY;
    for (int c = 0; c < nch; ++c) {
      const uint32_t slot = (used + c) % kRingSlots, ph = ((used + c) / kRingSlots) & 1;
      if (lane == 0 && c + 2 < nch) issue(c + 2);  // slot (c + 2) % 3 was released by the __syncwarp below
      mbar_wait(&full[slot], ph);
      const int nv = static_cast<int>(min(static_cast<int64_t>(kRingChunk / 16), nvec - static_cast<int64_t>(c) * (kRingChunk / 16)));
      const uint32_t sbase = smem_u32(ring + slot * kRingChunk);
      for (int b = 0; b < nv; b += 32) {  // warp-uniform trip count
        const int vi = b + lane;
        uint4 w = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
        if (vi < nv) {
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                       : "r"(sbase + vi * 16));
          bad |= nonfinite8(w);
        }
        const float gm = vi < nv ? max8(w) : -INFINITY;
        if (c == 0 && b == 0) floor = warp_kth_largest(gm, k);
        const bool h = vi < nv && gm >= fmaxf(floor, L.thr_v);
        if (__any_sync(0xffffffffu, h))
          offer_vectors(L, h, w, c0 + (static_cast<int64_t>(c) * (kRingChunk / 16) + vi) * 8, floor);
      }
      __syncwarp();  // every lane is done with this slot before lane 0 refills it
    }
    used += nch;
    // scalar tail of the segment (the V_local % 8 columns of the row's last segment)
    const uint16_t* T = p.T + static_cast<int64_t>(row) * p.ldT;
    for (int64_t cb = c0 + nvec * 8; cb < c1; cb += 32) {
      const int64_t col = cb + lane;
      float v = -INFINITY;
      if (col < c1) {
        const uint32_t b16 = T[col];
        bad |= static_cast<uint32_t>((b16 & 0x7FFFu) >= 0x7F80u);
        v = __uint_as_float(b16 << 16);
      }
      uint32_t hit = __ballot_sync(0xffffffffu, col < c1 && v >= floor && L.admits(v, static_cast<int32_t>(col)));
      while (hit) {
        const int s2 = __ffs(hit) - 1;
        hit &= hit - 1;
        L.offer(v, static_cast<int32_t>(col), s2);
      }
    }
    if (lane < k) {
      const int64_t o = (static_cast<int64_t>(row) * p.nseg + seg) * k;
      p.cand_val[o + lane] = L.v;
      p.cand_idx[o + lane] = (L.i == INT32_MAX) ? INT32_MAX : static_cast<int32_t>(L.i + p.vocab_offset);
    }
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (bad && lane == 0) atomicOr(p.lab.status, AURORA_STATUS_NONFINITE);
}

// --------------------------------------------------------------------------- A2 merge
// warp per row: merge `nlists` sorted lists of length k -> top list + argmax.  Up to 32 lists: a
// k-way merge, lane l holding the head of list l; each of the k steps picks the best head by
// (value desc, index asc) with a warp reduction and advances that list (k steps of ~20
// instructions instead of nlists * k list insertions).  The lists hold distinct indices.
__global__ void __launch_bounds__(256) k_topk_merge(VerifyLaunch p, const float* in_val, const int32_t* in_idx,
                                                    int nlists, int64_t row_stride, int64_t list_stride) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= p.M) return;
  const int k = p.k_max;
  if (nlists <= 32) {
    const int64_t base = static_cast<int64_t>(row) * row_stride + lane * list_stride;
    int pos = 0;
    float hv = -INFINITY;
    int32_t hi = INT32_MAX;
    if (lane < nlists) { hv = in_val[base]; hi = in_idx[base]; }
    float ov = -INFINITY;
    int32_t oi = INT32_MAX;
    for (int r = 0; r < k; ++r) {
      float bv = hv;
      int32_t bi = hi;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const float v2 = __shfl_xor_sync(0xffffffffu, bv, off);
        const int32_t i2 = __shfl_xor_sync(0xffffffffu, bi, off);
        if (better(v2, i2, bv, bi)) { bv = v2; bi = i2; }
      }
      if (lane == r) { ov = bv; oi = bi; }
      if (hv == bv && hi == bi && lane < nlists) {  // this lane's list supplied the winner: advance
        ++pos;
        if (pos < k) { hv = in_val[base + pos]; hi = in_idx[base + pos]; }
        else { hv = -INFINITY; hi = INT32_MAX; }
      }
    }
    if (lane < k) {
      p.top_val[static_cast<int64_t>(row) * k + lane] = ov;
      p.top_idx[static_cast<int64_t>(row) * k + lane] = oi;
    }
    const int32_t am = __shfl_sync(0xffffffffu, oi, 0);
    if (lane == 0) p.lab.target_argmax[row] = am;
    return;
  }
  WarpList F;
  F.init(k);
  for (int l = 0; l < nlists; ++l) {
    const int64_t o = static_cast<int64_t>(row) * row_stride + l * list_stride;
    const float cv = lane < k ? in_val[o + lane] : -INFINITY;
    const int32_t ci = lane < k ? in_idx[o + lane] : INT32_MAX;
    uint32_t hit = __ballot_sync(0xffffffffu, lane < k && F.admits(cv, ci));
    while (hit) {
      const int s = __ffs(hit) - 1;
      hit &= hit - 1;
      F.offer(cv, ci, s);
    }
  }
  if (lane < k) {
    p.top_val[static_cast<int64_t>(row) * k + lane] = F.v;
    p.top_idx[static_cast<int64_t>(row) * k + lane] = F.i;
  }
  const int32_t am = __shfl_sync(0xffffffffu, F.i, 0);
  if (lane == 0) p.lab.target_argmax[row] = am;
}

// --------------------------------------------------------------------------- A2' sparse
// NEXT F1: the target arrives as its top-K_t logits per row, (global id, bf16 logit)
// pairs in any order ("top-K logits filtering (e.g., K=1024)").  Warp per row:
// lanes stride over the pairs, the warp list keeps the top-k_max by (value desc, id asc).
// Status bits: non-finite logit, id outside [0, V), an id appearing twice in the top list.
__global__ void __launch_bounds__(256) k_target_scan_topk(VerifyLaunch p, const int32_t* __restrict__ tk_idx,
                                                          const uint16_t* __restrict__ tk_val, int32_t K_t) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= p.M) return;
  const int k = p.k_max;
  WarpList L;
  L.init(k);
  uint32_t err = 0;
  const int64_t o = static_cast<int64_t>(row) * K_t;
  for (int j0 = 0; j0 < K_t; j0 += 32) {
    const int j = j0 + lane;
    float v = -INFINITY;
    int32_t id = INT32_MAX;
    bool ok = false;
    if (j < K_t) {
      const uint32_t b = tk_val[o + j];
      id = tk_idx[o + j];
      if ((b & 0x7FFFu) >= 0x7F80u) err |= AURORA_STATUS_NONFINITE;
      else if (id < 0 || static_cast<int64_t>(id) >= p.V) err |= AURORA_STATUS_RANGE;
      else { v = __uint_as_float(b << 16); ok = true; }
    }
    uint32_t hit = __ballot_sync(0xffffffffu, ok && L.admits(v, id));
    while (hit) {
      const int src = __ffs(hit) - 1;
      hit &= hit - 1;
      const float cv = __shfl_sync(0xffffffffu, v, src);
      const int32_t ci = __shfl_sync(0xffffffffu, id, src);
      if (L.admits(cv, ci)) {
        if (__any_sync(0xffffffffu, lane < k && L.i == ci)) err |= AURORA_STATUS_STRUCTURE;  // duplicate id
        else L.insert(cv, ci);
      }
    }
  }
  err = __reduce_or_sync(0xffffffffu, err);
  if (lane < k) {
    p.top_val[static_cast<int64_t>(row) * k + lane] = L.v;
    p.top_idx[static_cast<int64_t>(row) * k + lane] = L.i;
  }
  const int32_t am = __shfl_sync(0xffffffffu, L.i, 0);
  if (lane == 0) {
    p.lab.target_argmax[row] = am;
    if (err) atomicOr(p.lab.status, err);
  }
}

// --------------------------------------------------------------------------- A3 verify
// warp per request; lane n = draft node n.
__global__ void __launch_bounds__(256) k_verify(VerifyLaunch p) {
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int n = threadIdx.x & 31;
  if (r >= p.R) return;
  const int N = p.N;
  const int nn = p.num_nodes ? min(max(p.num_nodes[r], 0), N) : N;
  const bool valid = n < nn;
  const int64_t base = static_cast<int64_t>(r) * (N + 1);
  uint32_t err = 0;
  int par = -1;
  int tok = -1;
  bool match = false;
  if (valid) {
    par = p.parents ? p.parents[static_cast<int64_t>(r) * N + n] : n - 1;
    if (par < -1 || par >= n) { err |= AURORA_STATUS_STRUCTURE; par = -1; }
    tok = p.draft[static_cast<int64_t>(r) * N + n];
    if (tok < 0 || static_cast<int64_t>(tok) >= p.V) err |= AURORA_STATUS_RANGE;
    match = (tok == p.lab.target_argmax[base + par + 1]);
  }
  // lowest-index sibling wins (reading Q12): drop a match if a lower sibling matched
  const uint32_t mball = __ballot_sync(0xffffffffu, match);
  bool blocked = false;
  for (int s = 0; s < 32; ++s) {
    const int ps = __shfl_sync(0xffffffffu, par, s);
    if (s < n && ((mball >> s) & 1u) && ps == par) blocked = true;
  }
  bool acc = valid && match && !blocked;
  // pointer jumping: acc &= acc[anc]; depth += depth[anc]
  int anc = valid ? par : -1;
  int depth = valid ? 1 : 0;
#pragma unroll
  for (int round = 0; round < 5; ++round) {
    const int src = anc >= 0 ? anc : n;
    const bool acc_a = __shfl_sync(0xffffffffu, acc, src);
    const int dep_a = __shfl_sync(0xffffffffu, depth, src);
    const int anc_a = __shfl_sync(0xffffffffu, anc, src);
    if (anc >= 0) {
      acc = acc && acc_a;
      depth += dep_a;
      anc = anc_a;
    }
  }
  const uint32_t accb = __ballot_sync(0xffffffffu, acc);
  const int a = __popc(accb);
  // deepest accepted node: depth == a
  const uint32_t deep = __ballot_sync(0xffffffffu, acc && depth == a);
  const int deepest_row = deep ? (__ffs(deep) - 1) + 1 : 0;
  // first-divergence flag for discard_scope 1: rejected node whose parent is accepted/root
  const bool par_acc = (par < 0) ? true : ((accb >> par) & 1u);
  uint8_t cls = AURORA_ROW_PAD;
  if (valid) {
    if (acc) cls = AURORA_ROW_ACCEPT;
    else if (p.cfg.discard_scope == 0 || par_acc) cls = AURORA_ROW_DISCARD;
  }
  if (n < N) {
    p.lab.accepted[static_cast<int64_t>(r) * N + n] = acc ? 1 : 0;
    p.lab.row_class[base + n + 1] = cls;
  }
  const uint32_t nacc = __popc(__ballot_sync(0xffffffffu, n < N && cls == AURORA_ROW_ACCEPT));
  const uint32_t ndis = __popc(__ballot_sync(0xffffffffu, n < N && cls == AURORA_ROW_DISCARD));
  err = __reduce_or_sync(0xffffffffu, err);
  if (n == 0) {
    p.lab.row_class[base] = AURORA_ROW_ACCEPT;
    p.lab.accept_len[r] = a + 1;
    p.lab.bonus[r] = p.lab.target_argmax[base + deepest_row];
    atomicAdd(&p.lab.counts[0], static_cast<int>(nacc) + 1);
    if (ndis) atomicAdd(&p.lab.counts[1], static_cast<int>(ndis));
    if (err) atomicOr(p.lab.status, err);
  }
}

// --------------------------------------------------------------------------- A4 finalize
// warp per row: lane j holds support entry j (k <= 16 <= 32); sums over a fixed xor tree
// (deterministic); the index-sorted order is each entry's rank among the row's ids.
__global__ void __launch_bounds__(256) k_finalize(VerifyLaunch p) {
  const int64_t m = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (m >= p.M) return;
  const int km = p.k_max;
  const uint8_t cls = p.lab.row_class[m];
  const int na = p.lab.counts[0], nd = p.lab.counts[1];
  int k = 0;
  float w = 0.f;
  if (cls == AURORA_ROW_ACCEPT) {
    k = p.cfg.k_accept;
    w = p.cfg.normalize ? 1.f / static_cast<float>(na + nd) : 1.f / static_cast<float>(na);
  } else if (cls == AURORA_ROW_DISCARD) {
    k = p.cfg.k_discard;
    w = p.cfg.normalize ? p.cfg.lambda_discard / static_cast<float>(na + nd)
                        : (nd > 0 ? p.cfg.lambda_discard / static_cast<float>(nd) : 0.f);
  }
  // F2: reverse-KL ACCEPT rows carry the support {y: beta} (the NTP term; the KL itself is
  // computed from T in the GEMM epilogues), dense-KL DISCARD rows an empty support with
  // H = E_p[t] - lse_t (sum_j p_j log p_j of the full target row).
  const bool f2_rkl = cls == AURORA_ROW_ACCEPT && p.cfg.accept_loss == 1;
  const bool f2_dense = cls == AURORA_ROW_DISCARD && p.cfg.k_discard == 0;
  if (f2_rkl || f2_dense) {
    const bool one = f2_rkl && p.cfg.ntp_beta > 0.f;
    for (int j = lane; j < km; j += 32) {
      p.lab.sup_idx[m * km + j] = (one && j == 0) ? p.top_idx[m * km] : INT32_MAX;
      p.lab.sup_p[m * km + j] = (one && j == 0) ? p.cfg.ntp_beta : 0.f;
    }
    if (lane == 0) {
      p.lab.row_H[m] = f2_dense ? p.ept[m] - p.lab.row_lse_t[m] : 0.f;
      p.lab.row_w[m] = w;
    }
    return;
  }
  const bool in = lane < k;
  const float v = in ? p.top_val[m * km + lane] : -INFINITY;
  const int32_t ix = in ? p.top_idx[m * km + lane] : INT32_MAX;
  const float t0 = __shfl_sync(0xffffffffu, v, 0);  // the row's largest (value-ordered list)
  float e = in ? expf(v - t0) : 0.f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  const float lz = logf(e);
  const float lp = v - t0 - lz;
  const float pj = in ? expf(lp) : 0.f;
  float h = in ? pj * lp : 0.f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  int rank = 0;  // position in the index-sorted support (ids are distinct)
  for (int i = 0; i < k; ++i) rank += (__shfl_sync(0xffffffffu, ix, i) < ix) ? 1 : 0;
  if (in) {
    p.lab.sup_idx[m * km + rank] = ix;
    p.lab.sup_p[m * km + rank] = pj;
  }
  for (int j = k + lane; j < km; j += 32) {
    p.lab.sup_idx[m * km + j] = INT32_MAX;
    p.lab.sup_p[m * km + j] = 0.f;
  }
  if (lane == 0) {
    p.lab.row_H[m] = k <= 1 ? 0.f : h;
    p.lab.row_w[m] = w;
  }
}

// --------------------------------------------------------------------------- F1 long supports
// Soft distillation over the transmitted top-K (k up to AURORA_MAX_K_SPARSE):
// the support of a row can hold every transmitted pair, too long for a warp list.  CTA
// per row: a block-wide bitonic sort of 64-bit keys in shared memory.
namespace {
// monotone float -> uint32 (numeric order, -0 == +0); finite inputs only
__device__ __forceinline__ uint32_t f2key(float v) {
  const uint32_t u = __float_as_uint(v == 0.f ? 0.f : v);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}
__device__ __forceinline__ int pow2_ceil(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}
// ascending bitonic sort of n (power of two) keys in smem; all threads of the block call it
__device__ void block_bitonic_sort(uint64_t* a, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < (n >> 1); t += blockDim.x) {
        const int lo = 2 * stride * (t / stride) + (t % stride);
        const int hi = lo + stride;
        const uint64_t x = a[lo], y = a[hi];
        if ((x > y) == ((lo & size) == 0)) { a[lo] = y; a[hi] = x; }
      }
    }
  }
  __syncthreads();
}
// deterministic block sum (fixed strided partials, fixed shuffle tree, warps in order)
__device__ float block_sum(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) t += red[i];
  return t;
}
}  // namespace

// A2' (long): sort the K_t pairs of a row by (value desc, id asc) -> top list [k_top],
// argmax; status bits as k_target_scan_topk (duplicate ids among the top k_top).
__global__ void __launch_bounds__(256) k_sort_pairs(VerifyLaunch p, const int32_t* __restrict__ tk_idx,
                                                    const uint16_t* __restrict__ tk_val, int32_t K_t) {
  extern __shared__ uint64_t keys[];
  __shared__ uint32_t s_err;
  const int64_t row = blockIdx.x;
  const int n = pow2_ceil(K_t);
  const int kt = p.k_top;
  if (threadIdx.x == 0) s_err = 0;
  uint32_t err = 0;
  const int64_t o = row * K_t;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    uint64_t key = ~0ull;
    if (j < K_t) {
      const uint32_t b = tk_val[o + j];
      const int32_t id = tk_idx[o + j];
      if ((b & 0x7FFFu) >= 0x7F80u) err |= AURORA_STATUS_NONFINITE;
      else if (id < 0 || static_cast<int64_t>(id) >= p.V) err |= AURORA_STATUS_RANGE;
      else key = (static_cast<uint64_t>(~f2key(__uint_as_float(b << 16))) << 32) | static_cast<uint32_t>(id);
    }
    keys[j] = key;
  }
  block_bitonic_sort(keys, n);
  for (int j = threadIdx.x; j < kt; j += blockDim.x) {
    const uint64_t key = keys[j];
    const bool valid = key != ~0ull;
    p.top_val[row * kt + j] = valid ? key2f(~static_cast<uint32_t>(key >> 32)) : -INFINITY;
    p.top_idx[row * kt + j] = valid ? static_cast<int32_t>(static_cast<uint32_t>(key)) : INT32_MAX;
  }
  if (threadIdx.x == 0)
    p.lab.target_argmax[row] = keys[0] != ~0ull ? static_cast<int32_t>(static_cast<uint32_t>(keys[0])) : INT32_MAX;
  // duplicate ids among the top kt: sort their ids, compare neighbours
  const int n2 = pow2_ceil(kt);
  __syncthreads();
  for (int j = threadIdx.x; j < n2; j += blockDim.x) {
    const uint64_t key = keys[j];
    keys[j] = (j < kt && key != ~0ull) ? static_cast<uint64_t>(static_cast<uint32_t>(key)) : ~0ull;
  }
  block_bitonic_sort(keys, n2);
  for (int j = threadIdx.x; j + 1 < kt; j += blockDim.x)
    if (keys[j] != ~0ull && keys[j] == keys[j + 1]) err |= AURORA_STATUS_STRUCTURE;
  if (err) atomicOr(&s_err, err);
  __syncthreads();
  if (threadIdx.x == 0 && s_err) atomicOr(p.lab.status, s_err);
}

// A4 (long): support = first k entries of the row's value-sorted top list, p~ =
// softmax of their logits (Eq. 3 target renormalised on S), H~ = sum p~ log p~, sorted by
// global id for the GEMM epilogues' merge-join.
__global__ void __launch_bounds__(256) k_finalize_long(VerifyLaunch p) {
  extern __shared__ uint64_t keys[];
  __shared__ float red[8];
  const int64_t m = blockIdx.x;
  const int km = p.k_max, kt = p.k_top;
  const uint8_t cls = p.lab.row_class[m];
  const int na = p.lab.counts[0], nd = p.lab.counts[1];
  int k = 0;
  float w = 0.f;
  if (cls == AURORA_ROW_ACCEPT) {
    k = p.cfg.k_accept;
    w = p.cfg.normalize ? 1.f / static_cast<float>(na + nd) : 1.f / static_cast<float>(na);
  } else if (cls == AURORA_ROW_DISCARD) {
    k = p.cfg.k_discard;
    w = p.cfg.normalize ? p.cfg.lambda_discard / static_cast<float>(na + nd)
                        : (nd > 0 ? p.cfg.lambda_discard / static_cast<float>(nd) : 0.f);
  }
  const float* tv = p.top_val + m * kt;
  const int32_t* ti = p.top_idx + m * kt;
  const float t0 = k > 0 ? tv[0] : 0.f;
  float e = 0.f;
  for (int j = threadIdx.x; j < k; j += blockDim.x) e += expf(tv[j] - t0);
  const float lz = logf(block_sum(e, red));
  const int n2 = pow2_ceil(k);
  float h = 0.f;
  for (int j = threadIdx.x; j < n2; j += blockDim.x) {
    uint64_t key = ~0ull;
    if (j < k) {
      const float lp = tv[j] - t0 - lz;
      const float pj = expf(lp);
      h += pj * lp;
      key = (static_cast<uint64_t>(static_cast<uint32_t>(ti[j])) << 32) | __float_as_uint(pj);
    }
    keys[j] = key;
  }
  float H = block_sum(h, red);
  if (k <= 1) H = 0.f;
  block_bitonic_sort(keys, n2);
  for (int j = threadIdx.x; j < km; j += blockDim.x) {
    const bool in = j < k;
    const uint64_t key = in ? keys[j] : 0ull;
    p.lab.sup_idx[m * km + j] = in ? static_cast<int32_t>(key >> 32) : INT32_MAX;
    p.lab.sup_p[m * km + j] = in ? __uint_as_float(static_cast<uint32_t>(key)) : 0.f;
  }
  if (threadIdx.x == 0) {
    p.lab.row_H[m] = H;
    p.lab.row_w[m] = w;
  }
}

// --------------------------------------------------------------------------- F2 row lse of T
// NEXT F2 (reverse KL / dense discard KL need p_target = softmax(T) over the full row):
// CTA per row, online (max, sum e^{t-m}, sum e^{t-m} t) over the row's vocab slice,
// deterministic merge (fixed strides, shuffle tree, warps in order).
__global__ void __launch_bounds__(256) k_row_lse_t(VerifyLaunch p) {
  const int64_t row = blockIdx.x;
  const uint16_t* tr = p.T + row * p.ldT;
  float m = -INFINITY, S = 0.f, A = 0.f;
  auto add = [&](float t) {
    if (t > m) {
      const float c = __expf(m - t);
      S *= c;
      A *= c;
      m = t;
    }
    const float e = __expf(t - m);
    S += e;
    A = fmaf(e, t, A);
  };
  for (int64_t j = threadIdx.x; j < p.V_local; j += blockDim.x) add(__uint_as_float(static_cast<uint32_t>(tr[j]) << 16));
  auto merge = [&](float m2, float S2, float A2) {
    const float mn = fmaxf(m, m2);
    if (mn == -INFINITY) return;
    const float a = __expf(m - mn), b = __expf(m2 - mn);
    S = S * a + S2 * b;
    A = A * a + A2 * b;
    m = mn;
  };
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, off);
    const float S2 = __shfl_xor_sync(0xffffffffu, S, off);
    const float A2 = __shfl_xor_sync(0xffffffffu, A, off);
    merge(m2, S2, A2);
  }
  __shared__ float red[3][8];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { red[0][w] = m; red[1][w] = S; red[2][w] = A; }
  __syncthreads();
  if (threadIdx.x == 0) {
    m = red[0][0]; S = red[1][0]; A = red[2][0];
    for (int i = 1; i < static_cast<int>(blockDim.x >> 5); ++i) merge(red[0][i], red[1][i], red[2][i]);
    if (p.lse_part) {  // vocab-parallel: this rank's (max, sum e^{t-m}, sum e^{t-m} t) for the allgather
      p.lse_part[row * 3 + 0] = m;
      p.lse_part[row * 3 + 1] = S;
      p.lse_part[row * 3 + 2] = A;
    } else {
      p.lab.row_lse_t[row] = m + logf(S);
      p.ept[row] = A / S;
    }
  }
}

// F2 x VP: merge the ranks' (max, sum e^{t-m}, sum e^{t-m} t) triples in rank order.
__global__ void __launch_bounds__(256) k_row_lse_t_combine(VerifyLaunch p, const float* __restrict__ parts, int P) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
  if (row >= p.M) return;
  float m = -INFINITY, S = 0.f, A = 0.f;
  for (int r = 0; r < P; ++r) {
    const float* q = parts + (static_cast<int64_t>(r) * p.M + row) * 3;
    const float mn = fmaxf(m, q[0]);
    if (mn == -INFINITY) continue;
    const float a = __expf(m - mn), b = __expf(q[0] - mn);
    S = S * a + q[1] * b;
    A = A * a + q[2] * b;
    m = mn;
  }
  p.lab.row_lse_t[row] = m + logf(S);
  p.ept[row] = A / S;
}

// --------------------------------------------------------------------------- launchers
cudaError_t launch_target_scan(const VerifyLaunch& p, cudaStream_t s) {
  k_target_scan<<<static_cast<unsigned>(p.M) * p.nseg, 256, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}
bool scan_ring_ok(const VerifyLaunch& p) {
  return (reinterpret_cast<uintptr_t>(p.T) & 15) == 0 && (p.ldT & 7) == 0 && (p.seg_len & 7) == 0;
}
int scan_ring_lists() { return 1; }
cudaError_t launch_target_scan_ring(const VerifyLaunch& p, cudaStream_t s) {
  constexpr int kSmem = kRingWarps * kRingSlots * kRingChunk + kRingWarps * kRingSlots * 8 + 128;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_target_scan_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int64_t items = static_cast<int64_t>(p.M) * p.nseg;
  const int64_t ctas = (items + kRingWarps - 1) / kRingWarps;
  const int grid = static_cast<int>(ctas < kNumSMs ? ctas : kNumSMs);
  k_target_scan_ring<<<grid, 32 * kRingWarps, kSmem, s>>>(p);
  count_launch();
  return cudaGetLastError();
}
bool scan_flat_ok(const VerifyLaunch& p) {
  return (p.V_local % 8) == 0 && (p.ldT % 8) == 0 && (reinterpret_cast<uintptr_t>(p.T) & 15) == 0;
}
int scan_flat_ctas() {
  static int c = [] {
    const char* e = getenv("AURORA_SCAN_FLAT_CTAS");
    return (e && atoi(e) == 3) ? 3 : kScanFlatCtas;
  }();
  return c;
}
FlatSplit flat_split(int64_t M, int64_t V_local) {
  FlatSplit f;
  f.V8 = V_local / 8;
  f.NV = M * f.V8;
  const int64_t warps = static_cast<int64_t>(scan_flat_ctas()) * kNumSMs * 8;
  f.W = static_cast<int32_t>(std::max<int64_t>(1, std::min<int64_t>(warps, f.NV / 64)));
  const int64_t minlen = std::max<int64_t>(1, f.NV / f.W);
  f.S = static_cast<int32_t>(std::min<int64_t>(f.W, (f.V8 + minlen - 1) / minlen + 1));
  return f;
}
int scan_flat_slots(int64_t M, int64_t V_local) { return flat_split(M, V_local).S; }
cudaError_t launch_target_scan_flat(const VerifyLaunch& p, int* nlists, cudaStream_t s) {
  const FlatSplit f = flat_split(p.M, p.V_local);
  *nlists = f.S;
  if (scan_flat_ctas() == 3)
    k_target_scan_flat<3><<<(f.W + 7) / 8, 256, 0, s>>>(p, f);
  else
    k_target_scan_flat<kScanFlatCtas><<<(f.W + 7) / 8, 256, 0, s>>>(p, f);
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_topk_merge(const VerifyLaunch& p, const float* in_val, const int32_t* in_idx, int nlists,
                              int64_t row_stride, int64_t list_stride, cudaStream_t s) {
  k_topk_merge<<<(p.M + 7) / 8, 256, 0, s>>>(p, in_val, in_idx, nlists, row_stride, list_stride);
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_target_scan_topk(const VerifyLaunch& p, const int32_t* tk_idx, const uint16_t* tk_val, int32_t K_t,
                                    cudaStream_t s) {
  k_target_scan_topk<<<(p.M + 7) / 8, 256, 0, s>>>(p, tk_idx, tk_val, K_t);
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_sort_pairs(const VerifyLaunch& p, const int32_t* tk_idx, const uint16_t* tk_val, int32_t K_t,
                              cudaStream_t s) {
  int n = 1;
  while (n < K_t) n <<= 1;
  const size_t smem = static_cast<size_t>(n) * sizeof(uint64_t);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_sort_pairs, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  k_sort_pairs<<<p.M, 256, smem, s>>>(p, tk_idx, tk_val, K_t);
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_finalize_long(const VerifyLaunch& p, cudaStream_t s) {
  int n = 1;
  while (n < p.k_top) n <<= 1;
  k_finalize_long<<<p.M, 256, static_cast<size_t>(n) * sizeof(uint64_t), s>>>(p);
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_row_lse_t(const VerifyLaunch& p, cudaStream_t s) {
  k_row_lse_t<<<p.M, 256, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_row_lse_t_combine(const VerifyLaunch& p, const float* parts, int P, cudaStream_t s) {
  k_row_lse_t_combine<<<(p.M + 255) / 256, 256, 0, s>>>(p, parts, P);
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_verify(const VerifyLaunch& p, cudaStream_t s) {
  k_verify<<<(p.R + 7) / 8, 256, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_finalize(const VerifyLaunch& p, cudaStream_t s) {
  k_finalize<<<(p.M + 7) / 8, 256, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace aur

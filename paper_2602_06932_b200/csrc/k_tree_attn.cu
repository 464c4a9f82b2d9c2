// k_tree_attn.cu — NEXT F4: tree attention of the draft layer, forward and backward.
//
// P:163-169 §3.2 "Efficient Tree Attention": one batched pass over every accepted and
// rejected branch with a mask that follows the speculative tree (parents[n] < n).
// Row s of request r (s = 0 root, s = n+1 draft node n) attends the P_r cached prefix
// positions of its request and the tree rows of its ancestor closure (F4-R1..R5).
//
// Default kernels when G (N+1) <= 128 (options tree_fwd_tc = 2, tree_bwd_tc = 1), tcgen05 / TMEM /
// TMA, persistent, work item = (request, kv head) with all its query rows as one M = 128 tile:
//   k_ta_fwd_tc2  two items in flight per SM (independent groups of TMA / MMA / 4 softmax warps),
//                 one-pass online softmax with lazy O rescaling in TMEM, P through shared memory.
//   k_ta_bwd_tc   one item per SM: S, dP, dV^T, dK^T, dQ MMAs from the TMA-loaded tiles into
//                 TMEM, P / dS in shared memory, dK / dV transposed through shared memory into
//                 whole 256 B key rows; 16 compute warps.
// Both take a warp-uniform unmasked path for prefix tiles wholly inside the request's prefix.
// The mma.sync kernels below are kept as options (and the split backward for G (N+1) > 128).
//
// mma.sync work decomposition (one launch per phase, no atomics, deterministic):
//   k_ta_fwd    CTA = (request, kv head, query-head chunk): the G query heads of a kv head
//               share every K/V tile they read (GQA), so a tile of 64 keys is loaded once for
//               up to 128 query rows = (heads x tree rows); warp = 16 query rows; online
//               softmax (FA2-style), K/V double-buffered through cp.async; O staged through
//               shared memory for 16-B stores; lse in natural log.
//   k_ta_dsum   warp per (row, head): Dsum = rowsum(dO * O) (fp32).
//   k_ta_bwd_dq the forward's decomposition: recompute S, P = exp(S - lse), dP = dO V^T,
//               dS = P (dP - Dsum), dQ += dS K (fp32 out).
//   k_ta_bwd_dkdv CTA = (128-key tile, kv head, request): 8 warps x 16 keys; every query
//               row of the request that can see the tile (all G heads x N+1 rows, streamed in
//               32-row chunks) is in the CTA, so dK/dV of a key are complete in one CTA and
//               are written once as bf16 — the G-head GQA sum happens in registers.
// mma.sync m16n8k16 bf16 (fp32 accumulate) with ldmatrix from 128-B-XOR swizzled shared tiles.
#include <cmath>
#include <initializer_list>
#include <type_traits>

#include "internal.h"
#include "ptx.cuh"

namespace aur {
namespace {

constexpr int D = 128;        // head dim
constexpr int ROWB = 2 * D;   // bytes per K/V/Q row
constexpr int KT2 = 128;      // keys per CTA (dK/dV kernel)
#ifndef TA_QC
#define TA_QC 32
#endif
constexpr int QC = TA_QC;     // query rows per streamed chunk (dK/dV kernel)
constexpr int kMaxRowsCta = 112;  // 7 warps: two CTAs per SM fit the register file
constexpr int kMaxRowsReq = 256;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

struct TaParams {
  const uint16_t *Q, *Kt, *Vt, *Kp, *Vp, *O, *dO;
  const float* lse;
  const float* Dsum;
  uint16_t* Oout;
  float* lse_out;
  float* dQ;
  uint16_t *dKt, *dVt, *dKp, *dVp;
  const int32_t *prefix_off, *parents, *num_nodes;
  uint32_t* status;
  int R, N, N1, Hq, Hkv, G, Gc, max_prefix;
  int prefix_total;  // rows of Kp / Vp; offsets beyond it are malformed
  float scale, c2;  // c2 = scale * log2(e)
};

__device__ __forceinline__ uint32_t swz(int row, int ch) { return row * ROWB + ((ch ^ (row & 7)) << 4); }
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

__device__ __forceinline__ void cp16(uint32_t s, const void* g, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int n>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(n) : "memory");
}
__device__ __forceinline__ void ldsm4(uint32_t (&r)[4], uint32_t a) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void ldsm4t(uint32_t (&r)[4], uint32_t a) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pk_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint4 lds_u4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}

// Prefix extent of request r: clamped to max_prefix; offsets outside [0, prefix_total] or
// decreasing make the request's prefix empty (its K/V are never read or written).  Either
// violation sets the RANGE bit when `flag`.
__device__ __forceinline__ void prefix_of(const TaParams& p, int r, int& p0, int& Pr, bool flag) {
  p0 = p.prefix_off[r];
  const int p1 = p.prefix_off[r + 1];
  int len = p1 - p0;
  if (p0 < 0 || len < 0 || p1 > p.prefix_total) {
    if (flag && p.status) atomicOr(p.status, (uint32_t)AURORA_STATUS_RANGE);
    p0 = 0;
    len = 0;
  } else if (len > p.max_prefix) {
    if (flag && p.status) atomicOr(p.status, (uint32_t)AURORA_STATUS_RANGE);
    len = p.max_prefix;
  }
  Pr = len;
}

// anc[s] (bit t = tree row t visible from row s), threads 0..N1-1.  0 = padded/malformed row.
__device__ void build_anc(const TaParams& p, int r, uint64_t* anc) {
  const int s = threadIdx.x;
  if (s >= p.N1) return;
  const int nn = p.num_nodes ? p.num_nodes[r] : p.N;
  bool bad = nn < 0 || nn > p.N;
  uint64_t m = 0;
  if (!bad) {
    if (s == 0) {
      m = 1ull;
    } else if (s - 1 < nn) {
      int cur = s - 1;
      m = 1ull | (1ull << s);
      for (int it = 0; it <= p.N; ++it) {
        const int par = p.parents ? p.parents[(size_t)r * p.N + cur] : cur - 1;
        if (par < -1 || par >= cur) { bad = true; break; }
        if (par < 0) break;
        m |= 1ull << (par + 1);
        cur = par;
      }
    }
  }
  if (bad && p.status) atomicOr(p.status, (uint32_t)AURORA_STATUS_STRUCTURE);
  anc[s] = bad ? 0ull : m;
}

__device__ __forceinline__ bool visible(uint64_t a, int kj, int Pr, int N1) {
  const int t = kj - Pr;
  return a != 0ull && (kj < Pr || (t < N1 && ((a >> t) & 1ull)));
}

// cp.async one K and one V tile of `nrows` keys starting at key0 (zero-filled past nkeys).
__device__ __forceinline__ void load_kv(const TaParams& p, uint32_t sK, uint32_t sV, int nrows, int key0, int nkeys,
                                        int Pr, int p0, int r, int hk) {
  for (int idx = threadIdx.x; idx < nrows * 16; idx += blockDim.x) {
    const int row = idx >> 4, ch = idx & 15, kj = key0 + row;
    const uint16_t *ks = p.Kt, *vs = p.Vt;
    int bytes = 0;
    if (kj < nkeys) {
      bytes = 16;
      size_t off;
      if (kj < Pr) {
        off = ((size_t)(p0 + kj) * p.Hkv + hk) * D + ch * 8;
        ks = p.Kp + off;
        vs = p.Vp + off;
      } else {
        off = (((size_t)r * p.N1 + (kj - Pr)) * p.Hkv + hk) * D + ch * 8;
        ks = p.Kt + off;
        vs = p.Vt + off;
      }
    }
    cp16(sK + swz(row, ch), ks, bytes);
    cp16(sV + swz(row, ch), vs, bytes);
  }
}

// cp.async query-ordered rows [i0, i0+nrows) of a [R, N1, Hq, D] tensor for heads h0.. into
// smem rows 0..nrows-1 (zero past `rows`).  Row i -> (g = i / N1, s = i % N1).
__device__ __forceinline__ void load_rows(const TaParams& p, const uint16_t* X, uint32_t sX, int i0, int nrows,
                                          int rows, int r, int h0) {
  for (int idx = threadIdx.x; idx < nrows * 16; idx += blockDim.x) {
    const int row = idx >> 4, ch = idx & 15, i = i0 + row;
    const uint16_t* src = X;
    int bytes = 0;
    if (i < rows) {
      const int g = i / p.N1, s = i - g * p.N1;
      src = X + (((size_t)r * p.N1 + s) * p.Hq + h0 + g) * D + ch * 8;
      bytes = 16;
    }
    cp16(sX + swz(row, ch), src, bytes);
  }
}

// S[16 x NK] (+)= A[16 rows of sA from arow0] . B[NK rows of sB]^T over D (both row-major).
template <int NK>
__device__ __forceinline__ void mma_rows_x_keys(float (&s)[NK / 8][4], uint32_t sA, int arow0, uint32_t sB, int lane) {
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    uint32_t a[4];
    ldsm4(a, sA + swz(arow0 + (lane & 7) + (((lane >> 3) & 1) << 3), 2 * ks + (lane >> 4)));
#pragma unroll
    for (int np = 0; np < NK / 16; ++np) {
      uint32_t b[4];
      ldsm4(b, sB + swz(np * 16 + (lane & 7) + ((lane >> 4) << 3), 2 * ks + ((lane >> 3) & 1)));
      mma16816(s[2 * np], a, b[0], b[1]);
      mma16816(s[2 * np + 1], a, b[2], b[3]);
    }
  }
}

// acc[16 x 128] += P[16 x NK] (C fragments, cast to bf16) . B[NK rows of sB, 128 cols].
template <int NK>
__device__ __forceinline__ void mma_p_x_rows(float (&acc)[16][4], const float (&pf)[NK / 8][4], uint32_t sB, int lane) {
#pragma unroll
  for (int kk = 0; kk < NK / 16; ++kk) {
    uint32_t a[4] = {pk_bf16(pf[2 * kk][0], pf[2 * kk][1]), pk_bf16(pf[2 * kk][2], pf[2 * kk][3]),
                     pk_bf16(pf[2 * kk + 1][0], pf[2 * kk + 1][1]), pk_bf16(pf[2 * kk + 1][2], pf[2 * kk + 1][3])};
#pragma unroll
    for (int np = 0; np < 8; ++np) {
      uint32_t b[4];
      ldsm4t(b, sB + swz(kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3), 2 * np + (lane >> 4)));
      mma16816(acc[2 * np], a, b[0], b[1]);
      mma16816(acc[2 * np + 1], a, b[2], b[3]);
    }
  }
}

// ------------------------------------------------------------------------------ forward
// K/V ring of ST stages x NK keys.  Every iteration commits exactly one cp.async group (possibly
// empty), so wait_group<ST-1> always means "tile t has landed".
template <int NK, int ST>
__device__ __forceinline__ void kv_prologue(const TaParams& p, uint32_t aK, uint32_t aV, int ntiles, int nkeys, int Pr,
                                            int p0, int r, int hk) {
#pragma unroll
  for (int j = 0; j < ST - 1; ++j) {
    if (j < ntiles) load_kv(p, aK + j * NK * ROWB, aV + j * NK * ROWB, NK, j * NK, nkeys, Pr, p0, r, hk);
    cp_commit();
  }
}
template <int NK, int ST>
__device__ __forceinline__ void kv_next(const TaParams& p, uint32_t aK, uint32_t aV, int t, int ntiles, int nkeys,
                                        int Pr, int p0, int r, int hk) {
  const int j = t + ST - 1;
  if (j < ntiles) load_kv(p, aK + (j % ST) * NK * ROWB, aV + (j % ST) * NK * ROWB, NK, j * NK, nkeys, Pr, p0, r, hk);
  cp_commit();
  cp_wait<ST - 1>();
  __syncthreads();
}

// One barrier per tile: wait for tile t, sync (so every warp is also done with tile t-1), then
// refill tile t-1's stage with tile t+ST-1.
template <int NK, int ST>
__device__ __forceinline__ void kv_next_1sync(const TaParams& p, uint32_t aK, uint32_t aV, int t, int ntiles,
                                              int nkeys, int Pr, int p0, int r, int hk) {
  cp_wait<ST - 2>();
  __syncthreads();
  const int j = t + ST - 1;
  if (j < ntiles) load_kv(p, aK + (j % ST) * NK * ROWB, aV + (j % ST) * NK * ROWB, NK, j * NK, nkeys, Pr, p0, r, hk);
  cp_commit();
}

// Raw scores of keys this warp's rows may not see -> -inf.  Skipped (warp-uniform) for tiles
// wholly inside the prefix when every row of the warp is a valid query row.
template <int NK>
__device__ __forceinline__ void mask_scores(float (&s)[NK / 8][4], bool fast, int key0, uint64_t a0, uint64_t a1,
                                            int Pr, int N1) {
  if (fast) return;
#pragma unroll
  for (int nt = 0; nt < NK / 8; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (!visible(e < 2 ? a0 : a1, key0 + nt * 8 + (e & 1), Pr, N1)) s[nt][e] = -INFINITY;
}

#ifndef TA_FWD_NK
#define TA_FWD_NK 64
#define TA_FWD_ST 2
#endif
constexpr int kFwdNK = TA_FWD_NK, kFwdST = TA_FWD_ST;

__global__ void __launch_bounds__(224, 2) k_ta_fwd(TaParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int NK = kFwdNK, ST = kFwdST;
  const int r = blockIdx.x, hk = blockIdx.y, hc = blockIdx.z;
  const int h0 = hk * p.G + hc * p.Gc;
  const int nh = min(p.Gc, p.G - hc * p.Gc);
  const int rows = nh * p.N1;
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + nw * 16 * ROWB;
  uint8_t* sV = sK + ST * NK * ROWB;
  uint64_t* anc = reinterpret_cast<uint64_t*>(sV + ST * NK * ROWB);
  const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aV = smem_u32(sV);

  int p0, Pr;
  prefix_of(p, r, p0, Pr, threadIdx.x == 0 && hk == 0 && hc == 0);
  const int nkeys = Pr + p.N1, ntiles = (nkeys + NK - 1) / NK;
  build_anc(p, r, anc);
  load_rows(p, p.Q, aQ, 0, nw * 16, rows, r, h0);
  kv_prologue<NK, ST>(p, aK, aV, ntiles, nkeys, Pr, p0, r, hk);  // Q rides in the first group

  const int i0 = warp * 16 + (lane >> 2), i1 = i0 + 8;
  uint64_t a0 = 0, a1 = 0;
  bool rows_ok = false;
  float o[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // m in scaled log2 units
  const float c2 = p.c2;

  for (int t = 0; t < ntiles; ++t) {
#ifdef TA_FWD_2SYNC
    kv_next<NK, ST>(p, aK, aV, t, ntiles, nkeys, Pr, p0, r, hk);
#else
    kv_next_1sync<NK, ST>(p, aK, aV, t, ntiles, nkeys, Pr, p0, r, hk);
#endif
    if (t == 0) {
      if (i0 < rows) a0 = anc[i0 % p.N1];
      if (i1 < rows) a1 = anc[i1 % p.N1];
      rows_ok = __all_sync(0xffffffffu, a0 != 0ull && a1 != 0ull);
    }
    const uint32_t kb = aK + (t % ST) * NK * ROWB, vb = aV + (t % ST) * NK * ROWB;
    float s[NK / 8][4];
#pragma unroll
    for (int j = 0; j < NK / 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
    mma_rows_x_keys<NK>(s, aQ, warp * 16, kb, lane);
    mask_scores<NK>(s, rows_ok && (t + 1) * NK <= Pr, t * NK + 2 * (lane & 3), a0, a1, Pr, p.N1);

    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < NK / 8; ++nt) {
      mx0 = fmaxf(mx0, fmaxf(s[nt][0], s[nt][1]));
      mx1 = fmaxf(mx1, fmaxf(s[nt][2], s[nt][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m0, mx0 * c2), mn1 = fmaxf(m1, mx1 * c2);
    const float ms0 = mn0 == -INFINITY ? 0.f : mn0, ms1 = mn1 == -INFINITY ? 0.f : mn1;
    const float al0 = ex2_approx(m0 - ms0), al1 = ex2_approx(m1 - ms1);  // m = -inf -> 0
    m0 = mn0;
    m1 = mn1;
    float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
    for (int nt = 0; nt < NK / 8; ++nt) {
      s[nt][0] = ex2_approx(fmaf(s[nt][0], c2, -ms0));
      s[nt][1] = ex2_approx(fmaf(s[nt][1], c2, -ms0));
      s[nt][2] = ex2_approx(fmaf(s[nt][2], c2, -ms1));
      s[nt][3] = ex2_approx(fmaf(s[nt][3], c2, -ms1));
      ls0 += s[nt][0] + s[nt][1];
      ls1 += s[nt][2] + s[nt][3];
    }
    l0 = l0 * al0 + ls0;
    l1 = l1 * al1 + ls1;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      o[j][0] *= al0;
      o[j][1] *= al0;
      o[j][2] *= al1;
      o[j][3] *= al1;
    }
    mma_p_x_rows<NK>(o, s, vb, lane);
#ifdef TA_FWD_2SYNC
    __syncthreads();
#endif
  }
  __syncthreads();  // the O staging below reuses sQ rows of this warp only, but K/V stages may refill

  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f, inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
  // stage the warp's 16 output rows (bf16) in its own rows of sQ, then 16-B stores
  const int lr0 = warp * 16 + (lane >> 2);
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) {
    sts32(aQ + swz(lr0, nt) + (lane & 3) * 4, pk_bf16(o[nt][0] * inv0, o[nt][1] * inv0));
    sts32(aQ + swz(lr0 + 8, nt) + (lane & 3) * 4, pk_bf16(o[nt][2] * inv1, o[nt][3] * inv1));
  }
  __syncwarp();
#pragma unroll
  for (int c = lane; c < 16 * 16; c += 32) {
    const int row = warp * 16 + (c >> 4), ch = c & 15;
    if (row < rows) {
      const int g = row / p.N1, s = row - g * p.N1;
      *reinterpret_cast<uint4*>(p.Oout + (((size_t)r * p.N1 + s) * p.Hq + h0 + g) * D + ch * 8) =
          lds_u4(aQ + swz(row, ch));
    }
  }
  if ((lane & 3) == 0) {
    if (i0 < rows) {
      const int g = i0 / p.N1, s = i0 - g * p.N1;
      p.lse_out[((size_t)r * p.N1 + s) * p.Hq + h0 + g] = l0 > 0.f ? (m0 + __log2f(l0)) * kLn2 : -INFINITY;
    }
    if (i1 < rows) {
      const int g = i1 / p.N1, s = i1 - g * p.N1;
      p.lse_out[((size_t)r * p.N1 + s) * p.Hq + h0 + g] = l1 > 0.f ? (m1 + __log2f(l1)) * kLn2 : -INFINITY;
    }
  }
}

// ------------------------------------------------------------------------------ backward
__global__ void __launch_bounds__(256) k_ta_dsum(const uint16_t* __restrict__ O, const uint16_t* __restrict__ dO,
                                                 float* __restrict__ Dsum, int64_t n_rows) {
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= n_rows) return;
  const uint2 o = *reinterpret_cast<const uint2*>(O + w * D + lane * 4);
  const uint2 g = *reinterpret_cast<const uint2*>(dO + w * D + lane * 4);
  const __nv_bfloat162* ob = reinterpret_cast<const __nv_bfloat162*>(&o);
  const __nv_bfloat162* gb = reinterpret_cast<const __nv_bfloat162*>(&g);
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const float2 a = __bfloat1622float2(ob[j]), b = __bfloat1622float2(gb[j]);
    acc += a.x * b.x + a.y * b.y;
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) Dsum[w] = acc;
}

constexpr int kDqNK = 32, kDqST = 3;

__global__ void __maxnreg__(144) k_ta_bwd_dq(TaParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int NK = kDqNK, ST = kDqST;
  const int r = blockIdx.x, hk = blockIdx.y, hc = blockIdx.z;
  const int h0 = hk * p.G + hc * p.Gc;
  const int nh = min(p.Gc, p.G - hc * p.Gc);
  const int rows = nh * p.N1;
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* sQ = smem;
  uint8_t* sdO = sQ + nw * 16 * ROWB;
  uint8_t* sK = sdO + nw * 16 * ROWB;
  uint8_t* sV = sK + ST * NK * ROWB;
  uint64_t* anc = reinterpret_cast<uint64_t*>(sV + ST * NK * ROWB);
  const uint32_t aQ = smem_u32(sQ), adO = smem_u32(sdO), aK = smem_u32(sK), aV = smem_u32(sV);

  int p0, Pr;
  prefix_of(p, r, p0, Pr, false);
  const int nkeys = Pr + p.N1, ntiles = (nkeys + NK - 1) / NK;
  build_anc(p, r, anc);
  load_rows(p, p.Q, aQ, 0, nw * 16, rows, r, h0);
  load_rows(p, p.dO, adO, 0, nw * 16, rows, r, h0);
  kv_prologue<NK, ST>(p, aK, aV, ntiles, nkeys, Pr, p0, r, hk);

  const int i0 = warp * 16 + (lane >> 2), i1 = i0 + 8;
  uint64_t a0 = 0, a1 = 0;
  bool rows_ok = false;
  float lse0 = 0.f, lse1 = 0.f, d0 = 0.f, d1 = 0.f;
  if (i0 < rows) {
    const int g = i0 / p.N1, s = i0 - g * p.N1;
    const size_t k = ((size_t)r * p.N1 + s) * p.Hq + h0 + g;
    lse0 = isinf(p.lse[k]) ? 0.f : p.lse[k] * kLog2e;  // padded rows: every key masked anyway
    d0 = p.Dsum[k];
  }
  if (i1 < rows) {
    const int g = i1 / p.N1, s = i1 - g * p.N1;
    const size_t k = ((size_t)r * p.N1 + s) * p.Hq + h0 + g;
    lse1 = isinf(p.lse[k]) ? 0.f : p.lse[k] * kLog2e;
    d1 = p.Dsum[k];
  }
  float dq[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j) dq[j][0] = dq[j][1] = dq[j][2] = dq[j][3] = 0.f;
  const float c2 = p.c2;

  for (int t = 0; t < ntiles; ++t) {
    kv_next<NK, ST>(p, aK, aV, t, ntiles, nkeys, Pr, p0, r, hk);
    if (t == 0) {
      if (i0 < rows) a0 = anc[i0 % p.N1];
      if (i1 < rows) a1 = anc[i1 % p.N1];
      rows_ok = __all_sync(0xffffffffu, a0 != 0ull && a1 != 0ull);
    }
    const uint32_t kb = aK + (t % ST) * NK * ROWB, vb = aV + (t % ST) * NK * ROWB;
    float s[NK / 8][4], dp[NK / 8][4];
#pragma unroll
    for (int j = 0; j < NK / 8; ++j) {
      s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
      dp[j][0] = dp[j][1] = dp[j][2] = dp[j][3] = 0.f;
    }
    mma_rows_x_keys<NK>(s, aQ, warp * 16, kb, lane);
    mma_rows_x_keys<NK>(dp, adO, warp * 16, vb, lane);
    mask_scores<NK>(s, rows_ok && (t + 1) * NK <= Pr, t * NK + 2 * (lane & 3), a0, a1, Pr, p.N1);
#pragma unroll
    for (int nt = 0; nt < NK / 8; ++nt) {
      s[nt][0] = ex2_approx(fmaf(s[nt][0], c2, -lse0)) * (dp[nt][0] - d0);  // dS (masked: exp2(-inf) = 0)
      s[nt][1] = ex2_approx(fmaf(s[nt][1], c2, -lse0)) * (dp[nt][1] - d0);
      s[nt][2] = ex2_approx(fmaf(s[nt][2], c2, -lse1)) * (dp[nt][2] - d1);
      s[nt][3] = ex2_approx(fmaf(s[nt][3], c2, -lse1)) * (dp[nt][3] - d1);
    }
    mma_p_x_rows<NK>(dq, s, kb, lane);  // dQ += dS K
    __syncthreads();
  }
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int i = half ? i1 : i0;
    if (i >= rows) continue;
    const int g = i / p.N1, s = i - g * p.N1;
    float* dst = p.dQ + (((size_t)r * p.N1 + s) * p.Hq + h0 + g) * D + 2 * (lane & 3);
#pragma unroll
    for (int nt = 0; nt < 16; ++nt)
      *reinterpret_cast<float2*>(dst + nt * 8) =
          make_float2(dq[nt][2 * half] * p.scale, dq[nt][2 * half + 1] * p.scale);
  }
}

__global__ void __launch_bounds__(256) k_ta_bwd_dkdv(TaParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tile = blockIdx.x, hk = blockIdx.y, r = blockIdx.z;
  int p0, Pr;
  prefix_of(p, r, p0, Pr, false);
  const int nkeys = Pr + p.N1, key0 = tile * KT2;
  if (key0 >= nkeys) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rows = p.G * p.N1, nchunks = (rows + QC - 1) / QC;
  uint8_t* sK = smem;
  uint8_t* sV = sK + KT2 * ROWB;
  uint8_t* sQ = sV + KT2 * ROWB;        // 2 stages x QC rows
  uint8_t* sdO = sQ + 2 * QC * ROWB;    // 2 stages x QC rows
  uint64_t* anc = reinterpret_cast<uint64_t*>(sdO + 2 * QC * ROWB);  // [40]
  uint64_t* ancr = anc + 40;                                          // [kMaxRowsReq]
  float* lse2 = reinterpret_cast<float*>(ancr + kMaxRowsReq);
  float* dsum = lse2 + kMaxRowsReq;
  int* chunk_ok = reinterpret_cast<int*>(dsum + kMaxRowsReq);  // [kMaxRowsReq / QC]
  const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aQ = smem_u32(sQ), adO = smem_u32(sdO);
  const int h0 = hk * p.G;

  build_anc(p, r, anc);
  load_kv(p, aK, aV, KT2, key0, nkeys, Pr, p0, r, hk);
  load_rows(p, p.Q, aQ, 0, QC, rows, r, h0);
  load_rows(p, p.dO, adO, 0, QC, rows, r, h0);
  cp_commit();
  __syncthreads();  // anc visible
  for (int i = threadIdx.x; i < nchunks * QC; i += blockDim.x) {
    uint64_t a = 0;
    float l = 0.f, dd = 0.f;
    if (i < rows) {
      const int g = i / p.N1, s = i - g * p.N1;
      const size_t k = ((size_t)r * p.N1 + s) * p.Hq + h0 + g;
      a = anc[s];
      l = p.lse[k] * kLog2e;
      dd = p.Dsum[k];
    }
    ancr[i] = a;
    lse2[i] = isinf(l) ? 0.f : l;
    dsum[i] = dd;
  }
  for (int c = warp; c < nchunks; c += blockDim.x >> 5) {  // chunk_ok[c]: all QC rows valid
    const int i = c * QC + lane;
    const bool v = __all_sync(0xffffffffu, lane >= QC || (i < rows && anc[i % p.N1] != 0ull));
    if (lane == 0) chunk_ok[c] = v ? 1 : 0;
  }

  float dv[16][4], dk[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    dv[j][0] = dv[j][1] = dv[j][2] = dv[j][3] = 0.f;
    dk[j][0] = dk[j][1] = dk[j][2] = dk[j][3] = 0.f;
  }
  const int kw = warp * 16;                       // this warp's keys within the tile
  const int kj0 = key0 + kw + (lane >> 2), kj1 = kj0 + 8;

  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) {
      const int st = (c + 1) & 1;
      load_rows(p, p.Q, aQ + st * QC * ROWB, (c + 1) * QC, QC, rows, r, h0);
      load_rows(p, p.dO, adO + st * QC * ROWB, (c + 1) * QC, QC, rows, r, h0);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const uint32_t qb = aQ + (c & 1) * QC * ROWB, gb = adO + (c & 1) * QC * ROWB;
    // S^T [16 keys x 32 rows] = K_w Q^T ; dP^T = V_w dO^T
    float s[QC / 8][4], dp[QC / 8][4];
#pragma unroll
    for (int j = 0; j < QC / 8; ++j) {
      s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
      dp[j][0] = dp[j][1] = dp[j][2] = dp[j][3] = 0.f;
    }
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      uint32_t ak[4], av[4];
      const int arow = kw + (lane & 7) + (((lane >> 3) & 1) << 3), ach = 2 * ks + (lane >> 4);
      ldsm4(ak, aK + swz(arow, ach));
      ldsm4(av, aV + swz(arow, ach));
#pragma unroll
      for (int np = 0; np < QC / 16; ++np) {
        uint32_t b[4];
        const int brow = np * 16 + (lane & 7) + ((lane >> 4) << 3), bch = 2 * ks + ((lane >> 3) & 1);
        ldsm4(b, qb + swz(brow, bch));
        mma16816(s[2 * np], ak, b[0], b[1]);
        mma16816(s[2 * np + 1], ak, b[2], b[3]);
        ldsm4(b, gb + swz(brow, bch));
        mma16816(dp[2 * np], av, b[0], b[1]);
        mma16816(dp[2 * np + 1], av, b[2], b[3]);
      }
    }
    // P^T, dS^T (C layout: rows = keys kj0/kj1, cols = query rows)
    const int qcol = c * QC + 2 * (lane & 3);
    const bool fast = chunk_ok[c] && key0 + kw + 16 <= Pr;  // warp-uniform: no mask needed
    if (!fast) {
#pragma unroll
      for (int nt = 0; nt < QC / 8; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (!visible(ancr[qcol + nt * 8 + (e & 1)], e < 2 ? kj0 : kj1, Pr, p.N1)) s[nt][e] = -INFINITY;
    }
#pragma unroll
    for (int nt = 0; nt < QC / 8; ++nt) {
#pragma unroll
      for (int e2 = 0; e2 < 2; ++e2) {
        const int i = qcol + nt * 8 + e2;
        const float l = lse2[i], dd = dsum[i];
#pragma unroll
        for (int e = e2; e < 4; e += 2) {
          const float pv = ex2_approx(fmaf(s[nt][e], p.c2, -l));  // masked: exp2(-inf) = 0
          s[nt][e] = pv;
          dp[nt][e] = pv * (dp[nt][e] - dd);
        }
      }
    }
    // dV += P^T dO ; dK += dS^T Q   (k = the chunk's 32 query rows)
#pragma unroll
    for (int kk = 0; kk < QC / 16; ++kk) {
      const uint32_t ap[4] = {pk_bf16(s[2 * kk][0], s[2 * kk][1]), pk_bf16(s[2 * kk][2], s[2 * kk][3]),
                              pk_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]), pk_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3])};
      const uint32_t ad[4] = {pk_bf16(dp[2 * kk][0], dp[2 * kk][1]), pk_bf16(dp[2 * kk][2], dp[2 * kk][3]),
                              pk_bf16(dp[2 * kk + 1][0], dp[2 * kk + 1][1]),
                              pk_bf16(dp[2 * kk + 1][2], dp[2 * kk + 1][3])};
#pragma unroll
      for (int np = 0; np < 8; ++np) {
        uint32_t b[4];
        const int brow = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3), bch = 2 * np + (lane >> 4);
        ldsm4t(b, gb + swz(brow, bch));
        mma16816(dv[2 * np], ap, b[0], b[1]);
        mma16816(dv[2 * np + 1], ap, b[2], b[3]);
        ldsm4t(b, qb + swz(brow, bch));
        mma16816(dk[2 * np], ad, b[0], b[1]);
        mma16816(dk[2 * np + 1], ad, b[2], b[3]);
      }
    }
    __syncthreads();
  }
  // stage bf16 dK (scaled) / dV rows in sK / sV (every warp is past its last read), then 16-B stores
  const int lr = kw + (lane >> 2);
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) {
    sts32(aK + swz(lr, nt) + (lane & 3) * 4, pk_bf16(dk[nt][0] * p.scale, dk[nt][1] * p.scale));
    sts32(aK + swz(lr + 8, nt) + (lane & 3) * 4, pk_bf16(dk[nt][2] * p.scale, dk[nt][3] * p.scale));
    sts32(aV + swz(lr, nt) + (lane & 3) * 4, pk_bf16(dv[nt][0], dv[nt][1]));
    sts32(aV + swz(lr + 8, nt) + (lane & 3) * 4, pk_bf16(dv[nt][2], dv[nt][3]));
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < KT2 * 16; idx += blockDim.x) {
    const int row = idx >> 4, ch = idx & 15, kj = key0 + row;
    if (kj >= nkeys) continue;
    size_t off;
    uint16_t *dk_dst, *dv_dst;
    if (kj < Pr) {
      off = ((size_t)(p0 + kj) * p.Hkv + hk) * D + ch * 8;
      dk_dst = p.dKp;
      dv_dst = p.dVp;
    } else {
      off = (((size_t)r * p.N1 + (kj - Pr)) * p.Hkv + hk) * D + ch * 8;
      dk_dst = p.dKt;
      dv_dst = p.dVt;
    }
    *reinterpret_cast<uint4*>(dk_dst + off) = lds_u4(aK + swz(row, ch));
    *reinterpret_cast<uint4*>(dv_dst + off) = lds_u4(aV + swz(row, ch));
  }
}

// Fused backward for G*(N+1) <= 128 (every query row of (request, kv head) in one CTA): per
// 32-key tile, a row phase (warp = 16 query rows: S, dP, P, dS, dQ += dS K; P and dS parked in
// shared memory as bf16) and a key phase (warp = 16 keys x 32 head-dim columns: dV = P^T dO,
// dK = dS^T Q over all rows) -- the five backward products each run once, K/V are read once,
// and dK/dV of a tile are complete when the tile is done (stored once, no atomics).
#ifndef TA_FB_NK
#define TA_FB_NK 64
#endif
constexpr int kFbNK = TA_FB_NK, kFbST = 3;
constexpr int kFbRowB = kFbNK * 2;  // bytes per row of the parked P / dS tiles

__device__ __forceinline__ uint32_t swz_p(int row, int ch) {
  if constexpr (kFbRowB == 128) return row * 128 + ((ch ^ (row & 7)) << 4);
  else return row * kFbRowB + ((ch ^ ((row >> 1) & 3)) << 4);
}

__global__ void __launch_bounds__(256) k_ta_bwd_fused(TaParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int NK = kFbNK, ST = kFbST;
  const int r = blockIdx.x, hk = blockIdx.y;
  const int h0 = hk * p.G;
  const int rows = p.G * p.N1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* sQ = smem;                       // 128 rows
  uint8_t* sdO = sQ + 128 * ROWB;
  uint8_t* sK = sdO + 128 * ROWB;
  uint8_t* sV = sK + ST * NK * ROWB;
  uint8_t* sP = sV + ST * NK * ROWB;        // [128 rows][NK keys] bf16
  uint8_t* sdS = sP + 128 * kFbRowB;
  uint64_t* anc = reinterpret_cast<uint64_t*>(sdS + 128 * kFbRowB);
  const uint32_t aQ = smem_u32(sQ), adO = smem_u32(sdO), aK = smem_u32(sK), aV = smem_u32(sV);
  const uint32_t aP = smem_u32(sP), adS = smem_u32(sdS);

  int p0, Pr;
  prefix_of(p, r, p0, Pr, false);
  const int nkeys = Pr + p.N1, ntiles = (nkeys + NK - 1) / NK;
  build_anc(p, r, anc);
  load_rows(p, p.Q, aQ, 0, 128, rows, r, h0);
  load_rows(p, p.dO, adO, 0, 128, rows, r, h0);
  kv_prologue<NK, ST>(p, aK, aV, ntiles, nkeys, Pr, p0, r, hk);

  const int i0 = warp * 16 + (lane >> 2), i1 = i0 + 8;
  uint64_t a0 = 0, a1 = 0;
  bool rows_ok = false;
  float lse0 = 0.f, lse1 = 0.f, d0 = 0.f, d1 = 0.f;
  if (i0 < rows) {
    const int g = i0 / p.N1, s = i0 - g * p.N1;
    const size_t k = ((size_t)r * p.N1 + s) * p.Hq + h0 + g;
    lse0 = isinf(p.lse[k]) ? 0.f : p.lse[k] * kLog2e;
    d0 = p.Dsum[k];
  }
  if (i1 < rows) {
    const int g = i1 / p.N1, s = i1 - g * p.N1;
    const size_t k = ((size_t)r * p.N1 + s) * p.Hq + h0 + g;
    lse1 = isinf(p.lse[k]) ? 0.f : p.lse[k] * kLog2e;
    d1 = p.Dsum[k];
  }
  float dq[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j) dq[j][0] = dq[j][1] = dq[j][2] = dq[j][3] = 0.f;
  const float c2 = p.c2;
  const int nks = (rows + 15) >> 4;               // 16-row steps holding valid rows

  for (int t = 0; t < ntiles; ++t) {
    kv_next<NK, ST>(p, aK, aV, t, ntiles, nkeys, Pr, p0, r, hk);
    if (t == 0) {
      if (i0 < rows) a0 = anc[i0 % p.N1];
      if (i1 < rows) a1 = anc[i1 % p.N1];
      rows_ok = __all_sync(0xffffffffu, a0 != 0ull && a1 != 0ull);
    }
    const uint32_t kb = aK + (t % ST) * NK * ROWB, vb = aV + (t % ST) * NK * ROWB;
    // ---- row phase (warps past the last valid row have nothing to do)
    if (warp < nks) {
      float s[NK / 8][4], dp[NK / 8][4];
#pragma unroll
      for (int j = 0; j < NK / 8; ++j) {
        s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
        dp[j][0] = dp[j][1] = dp[j][2] = dp[j][3] = 0.f;
      }
      mma_rows_x_keys<NK>(s, aQ, warp * 16, kb, lane);
      mma_rows_x_keys<NK>(dp, adO, warp * 16, vb, lane);
      mask_scores<NK>(s, rows_ok && (t + 1) * NK <= Pr, t * NK + 2 * (lane & 3), a0, a1, Pr, p.N1);
      const int lr = warp * 16 + (lane >> 2);
#pragma unroll
      for (int nt = 0; nt < NK / 8; ++nt) {
        const float p0v = ex2_approx(fmaf(s[nt][0], c2, -lse0)), p1v = ex2_approx(fmaf(s[nt][1], c2, -lse0));
        const float p2v = ex2_approx(fmaf(s[nt][2], c2, -lse1)), p3v = ex2_approx(fmaf(s[nt][3], c2, -lse1));
        sts32(aP + swz_p(lr, nt) + (lane & 3) * 4, pk_bf16(p0v, p1v));
        sts32(aP + swz_p(lr + 8, nt) + (lane & 3) * 4, pk_bf16(p2v, p3v));
        s[nt][0] = p0v * (dp[nt][0] - d0);
        s[nt][1] = p1v * (dp[nt][1] - d0);
        s[nt][2] = p2v * (dp[nt][2] - d1);
        s[nt][3] = p3v * (dp[nt][3] - d1);
        sts32(adS + swz_p(lr, nt) + (lane & 3) * 4, pk_bf16(s[nt][0], s[nt][1]));
        sts32(adS + swz_p(lr + 8, nt) + (lane & 3) * 4, pk_bf16(s[nt][2], s[nt][3]));
      }
      mma_p_x_rows<NK>(dq, s, kb, lane);  // dQ += dS K
    }
    __syncthreads();
    // ---- key phase: warp = 32 keys (two 16-key m-tiles) x 32 head dims; dV = P^T dO, dK = dS^T Q
    // over the valid rows.  Each B fragment (dO, Q) now feeds two m-tiles: 8 ldmatrix per 16 MMAs.
    {
      static_assert(kFbNK == 64, "key phase tiling assumes 64-key tiles");
      const int kp = warp & 1, g32 = warp >> 1;
      float dv[2][4][4], dk[2][4][4];
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dv[m][j][0] = dv[m][j][1] = dv[m][j][2] = dv[m][j][3] = 0.f;
          dk[m][j][0] = dk[m][j][1] = dk[m][j][2] = dk[m][j][3] = 0.f;
        }
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {  // 16 query rows per step
        if (ks >= nks) break;
        uint32_t ap[2][4], ad[2][4];
        const int prow = ks * 16 + (lane & 7) + ((lane >> 4) << 3);
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          const int pch = 2 * (2 * kp + m) + ((lane >> 3) & 1);
          ldsm4t(ap[m], aP + swz_p(prow, pch));
          ldsm4t(ad[m], adS + swz_p(prow, pch));
        }
#pragma unroll
        for (int np = 0; np < 2; ++np) {
          uint32_t b[4];
          const int brow = ks * 16 + (lane & 7) + (((lane >> 3) & 1) << 3), bch = 4 * g32 + 2 * np + (lane >> 4);
          ldsm4t(b, adO + swz(brow, bch));
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            mma16816(dv[m][2 * np], ap[m], b[0], b[1]);
            mma16816(dv[m][2 * np + 1], ap[m], b[2], b[3]);
          }
          ldsm4t(b, aQ + swz(brow, bch));
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            mma16816(dk[m][2 * np], ad[m], b[0], b[1]);
            mma16816(dk[m][2 * np + 1], ad[m], b[2], b[3]);
          }
        }
      }
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int kj = t * NK + (2 * kp + m) * 16 + (lane >> 2) + half * 8;
          if (kj >= nkeys) continue;
          size_t off;
          uint16_t *dk_dst, *dv_dst;
          if (kj < Pr) {
            off = ((size_t)(p0 + kj) * p.Hkv + hk) * D;
            dk_dst = p.dKp;
            dv_dst = p.dVp;
          } else {
            off = (((size_t)r * p.N1 + (kj - Pr)) * p.Hkv + hk) * D;
            dk_dst = p.dKt;
            dv_dst = p.dVt;
          }
          off += 32 * g32 + 2 * (lane & 3);
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            *reinterpret_cast<uint32_t*>(dv_dst + off + nt * 8) = pk_bf16(dv[m][nt][2 * half], dv[m][nt][2 * half + 1]);
            *reinterpret_cast<uint32_t*>(dk_dst + off + nt * 8) =
                pk_bf16(dk[m][nt][2 * half] * p.scale, dk[m][nt][2 * half + 1] * p.scale);
          }
        }
    }

  }
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int i = half ? i1 : i0;
    if (i >= rows) continue;
    const int g = i / p.N1, s = i - g * p.N1;
    float* dst = p.dQ + (((size_t)r * p.N1 + s) * p.Hq + h0 + g) * D + 2 * (lane & 3);
#pragma unroll
    for (int nt = 0; nt < 16; ++nt)
      *reinterpret_cast<float2*>(dst + nt * 8) =
          make_float2(dq[nt][2 * half] * p.scale, dq[nt][2 * half + 1] * p.scale);
  }
}

// ------------------------------------------------------------------------------ tcgen05 forward
// Persistent, one CTA per SM, work item = (request, KV head) with all G*(N+1) <= 128 query rows
// of the KV head as the M = 128 rows of the UMMA tile.  Warp roles: warp 0 = TMA producer (Q box,
// then K / V tiles of 64 keys through a 4-stage ring: the request's prefix tiles from Kp/Vp, then
// one tree tile from Kt/Vt), warp 1 = MMA issuer (tcgen05.mma kind::f16, fp32 accumulators in
// TMEM), warps 2-9 = softmax (thread = TMEM lane = query row; warps w and w+4 split the 64 key
// columns of a tile).  Two passes over the key tiles per item: pass A accumulates the row max /
// sum-exp of S = Q K^T (S double-buffered in TMEM), pass B recomputes S, writes the normalised
// P = exp(S - lse) as bf16 into shared memory (the A operand, K-major SW128, double-buffered)
// and accumulates O += P V in TMEM (V as the MN-major B operand) — O is never rescaled.
// TMEM columns: S[0] 0..63, S[1] 64..127, O 128..255.
#ifdef TA_TC_SPIN
#define TC_WAIT mbar_wait
#else
#define TC_WAIT mbar_wait_sleep
#endif
struct TaTcMaps {
  CUtensorMap Q, Kp, Vp, Kt, Vt;
};
constexpr int kTcNK = 64;                     // keys per item
constexpr int kTcKST = 6;                     // K ring depth (released when S completes)
constexpr int kTcVST = 3;                     // V ring depth (released when P V completes)
constexpr int kTcNS = 4;                      // S buffers in TMEM (columns 0 .. 4*64), O after them
constexpr int kTcThreads = 320;               // TMA warp, MMA warp, 8 softmax warps
constexpr int kTcOffQ = 0;                    // 2 K-major atoms [128 rows x 128 B]
constexpr int kTcSlot = 2 * kTcNK * 128;      // 16 KB: K (2 atoms [64 x 128 B]) or V (2 MN slices)
constexpr int kTcOffK = 32768;
constexpr int kTcOffV = kTcOffK + kTcKST * kTcSlot;
constexpr int kTcOffP = kTcOffV + kTcVST * kTcSlot;
constexpr int kTcPBuf = 128 * kTcNK * 2;      // 16 KB: [128 rows x 64 keys] bf16, one K atom
constexpr int kTcOffBar = kTcOffP + 2 * kTcPBuf;
constexpr size_t kSmemTc = kTcOffBar + 512 + 4096 + 1024;  // barriers, anc, (m, l) exchange, align

// K-major SW128 operand with `rows` rows per 64-element K atom; k-step kk = 16 elements.
__device__ __forceinline__ uint64_t kmaj_desc(uint32_t base, int kk, int rows) {
  return umma_desc_sw128(base + (kk >> 2) * rows * 128 + (kk & 3) * 32, 16, 1024);
}
// MN-major SW128 B operand [K rows x 128 MN] stored as two 64-wide MN slices of `krows` rows.
__device__ __forceinline__ uint64_t mnmaj_desc(uint32_t base, int kk, int krows) {
  return umma_desc_sw128(base + kk * 2048, krows * 128, 1024);
}

__global__ void __launch_bounds__(kTcThreads, 1) k_ta_fwd_tc(const __grid_constant__ TaTcMaps maps, TaParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTcOffBar);
  uint64_t* q_full = bars + 0;
  uint64_t* q_free = bars + 1;
  uint64_t* k_full = bars + 2;    // [6]
  uint64_t* k_empty = bars + 8;   // [6]
  uint64_t* v_full = bars + 14;   // [3]
  uint64_t* v_empty = bars + 17;  // [3]
  uint64_t* s_full = bars + 20;   // [kTcNS]
  uint64_t* s_free = bars + 24;   // [kTcNS]
  uint64_t* p_full = bars + 28;   // [2]
  uint64_t* p_free = bars + 30;   // [2]
  uint64_t* o_done = bars + 32;
  uint64_t* o_free = bars + 33;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 34);
  uint64_t* anc = bars + 36;      // [40]
  const int G = p.G, N1 = p.N1;
  const int nwork = p.R * p.Hkv;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_free, 1);
    for (int s = 0; s < kTcKST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < kTcVST; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < kTcNS; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_free[s], 256);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&p_full[s], 256);
      mbar_init(&p_free[s], 1);
    }
    mbar_init(o_done, 1);
    mbar_init(o_free, 256);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&maps.Q);
      tma_prefetch_desc(&maps.Kp);
      tma_prefetch_desc(&maps.Vp);
      tma_prefetch_desc(&maps.Kt);
      tma_prefetch_desc(&maps.Vt);
      uint32_t ki = 0, vi = 0;  // global K / V load counters
      int wi = 0;
      for (int w = blockIdx.x; w < nwork; w += gridDim.x, ++wi) {
        const int r = w / p.Hkv, hk = w - r * p.Hkv;
        int p0, Pr;
        prefix_of(p, r, p0, Pr, hk == 0);
        const int npt = (Pr + kTcNK - 1) / kTcNK, ntiles = npt + 1;
        if (wi > 0) TC_WAIT(q_free, (wi - 1) & 1);
        mbar_arrive_expect_tx(q_full, 2u * 128u * G * N1);
        tma_load_3d(&maps.Q, q_full, smem + kTcOffQ, 0, hk * G, r * N1);
        tma_load_3d(&maps.Q, q_full, smem + kTcOffQ + 16384, 64, hk * G, r * N1);
        for (int it = 0; it < 2 * ntiles; ++it) {
          const int j = it % ntiles;
          const bool pass_b = it >= ntiles;
          const CUtensorMap* mk = j < npt ? &maps.Kp : &maps.Kt;
          const CUtensorMap* mv = j < npt ? &maps.Vp : &maps.Vt;
          const int z = j < npt ? p0 + j * kTcNK : r * N1;
          {
            const int ks = ki % kTcKST;
            if (ki >= kTcKST) TC_WAIT(&k_empty[ks], ((ki / kTcKST) & 1) ^ 1);
            uint8_t* kd = smem + kTcOffK + ks * kTcSlot;
#ifdef TA_TC_NOLOAD
            mbar_arrive(&k_full[ks]);
            (void)kd; (void)mk;
#else
            mbar_arrive_expect_tx(&k_full[ks], kTcSlot);
            tma_load_3d(mk, &k_full[ks], kd, 0, hk, z);
            tma_load_3d(mk, &k_full[ks], kd + kTcNK * 128, 64, hk, z);
#endif
            ++ki;
          }
          if (pass_b) {
            const int vs = vi % kTcVST;
            if (vi >= kTcVST) TC_WAIT(&v_empty[vs], ((vi / kTcVST) & 1) ^ 1);
            uint8_t* vd = smem + kTcOffV + vs * kTcSlot;
#ifdef TA_TC_NOLOAD
            mbar_arrive(&v_full[vs]);
            (void)vd; (void)mv;
#else
            mbar_arrive_expect_tx(&v_full[vs], kTcSlot);
            tma_load_3d(mv, &v_full[vs], vd, 0, hk, z);
            tma_load_3d(mv, &v_full[vs], vd + kTcNK * 128, 64, hk, z);
#endif
            ++vi;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = umma_idesc_bf16(128, kTcNK, false, false);
      constexpr uint32_t idPV = umma_idesc_bf16(128, 128, false, true);
      const uint32_t aQ = smem_u32(smem + kTcOffQ), aP = smem_u32(smem + kTcOffP);
      uint32_t gs = 0, pb = 0;  // S items issued (= K items consumed), P V items (= V items consumed)
      int wi = 0;
      for (int w = blockIdx.x; w < nwork; w += gridDim.x, ++wi) {
        const int r = w / p.Hkv;
        int p0, Pr;
        prefix_of(p, r, p0, Pr, false);
        const int ntiles = (Pr + kTcNK - 1) / kTcNK + 1, total = 2 * ntiles;
        TC_WAIT(q_full, wi & 1);
        auto issue_s = [&](uint32_t g) {
          const int ks = g % kTcKST, sb = g % kTcNS;
          TC_WAIT(&k_full[ks], (g / kTcKST) & 1);
          if (g >= kTcNS) TC_WAIT(&s_free[sb], ((g / kTcNS) & 1) ^ 1);
          tc_fence_after();
          const uint32_t kb = smem_u32(smem + kTcOffK + ks * kTcSlot);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16(tmem + sb * kTcNK, kmaj_desc(aQ, kk, 128), kmaj_desc(kb, kk, kTcNK), idS, kk > 0);
          umma_commit(&s_full[sb]);
          umma_commit(&k_empty[ks]);  // the K slot is free once this S has been computed
        };
        const uint32_t g0 = gs;  // S items run up to kTcNS - 1 ahead of the P V item
        for (int k = 0; k < kTcNS - 1 && k < total; ++k) issue_s(gs++);
        for (int it = 0; it < total; ++it) {
          if (it + kTcNS - 1 < total) issue_s(gs++);
          (void)g0;
          if (it >= ntiles) {
            const int jb = it - ntiles, pbuf = pb & 1, vs = pb % kTcVST;
            if (jb == 0 && wi > 0) TC_WAIT(o_free, (wi - 1) & 1);  // epilogue read the previous O
            TC_WAIT(&v_full[vs], (pb / kTcVST) & 1);
            TC_WAIT(&p_full[pbuf], (pb >> 1) & 1);
            tc_fence_after();
            const uint32_t vb = smem_u32(smem + kTcOffV + vs * kTcSlot);
#pragma unroll
            for (int kk = 0; kk < kTcNK / 16; ++kk)
              umma_bf16(tmem + kTcNS * kTcNK, kmaj_desc(aP + pbuf * kTcPBuf, kk, 128), mnmaj_desc(vb, kk, kTcNK), idPV,
                        (jb > 0 || kk > 0) ? 1u : 0u);
            umma_commit(&p_free[pbuf]);
            umma_commit(&v_empty[vs]);
            ++pb;
          }
        }
        umma_commit(o_done);
        umma_commit(q_free);
      }
    }
  } else {
    // ---- softmax / epilogue warps (8): thread = query row i (TMEM lane) x column half hf.
    const int q4 = warp & 3, hf = (warp - 2) >> 2;
    const int i = q4 * 32 + lane;
    const int rows = G * N1;
    const uint32_t trow = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
    const uint32_t aProw = smem_u32(smem + kTcOffP) + i * 128;
    float* stat = reinterpret_cast<float*>(anc + 40);  // [2 halves][2][128]: (m, l)
    const float c2 = p.c2;
    const int st_id = threadIdx.x - 64;                 // 0..255
    uint32_t gs = 0, pb = 0;
    int wi = 0;
    for (int w = blockIdx.x; w < nwork; w += gridDim.x, ++wi) {
      const int r = w / p.Hkv, hk = w - r * p.Hkv;
      int p0, Pr;
      prefix_of(p, r, p0, Pr, false);
      const int npt = (Pr + kTcNK - 1) / kTcNK, ntiles = npt + 1;
      if (st_id < N1) {  // ancestor masks of this request
        const int s = st_id;
        const int nn = p.num_nodes ? p.num_nodes[r] : p.N;
        bool bad = nn < 0 || nn > p.N;
        uint64_t m = 0;
        if (!bad) {
          if (s == 0) {
            m = 1ull;
          } else if (s - 1 < nn) {
            int cur = s - 1;
            m = 1ull | (1ull << s);
            for (int k = 0; k <= p.N; ++k) {
              const int par = p.parents ? p.parents[(size_t)r * p.N + cur] : cur - 1;
              if (par < -1 || par >= cur) { bad = true; break; }
              if (par < 0) break;
              m |= 1ull << (par + 1);
              cur = par;
            }
          }
        }
        if (bad && p.status && hk == 0) atomicOr(p.status, (uint32_t)AURORA_STATUS_STRUCTURE);
        anc[s] = bad ? 0ull : m;
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const int s_row = i / G, g = i - s_row * G;
      const uint64_t a = i < rows ? anc[s_row] : 0ull;
      const uint64_t ah = hf ? (a >> 32) : a;           // tree-tile bits of this half's 32 columns
      float m = -INFINITY, l = 0.f, mfin = 0.f;
      for (int it = 0; it < 2 * ntiles; ++it, ++gs) {
        const int sb = gs % kTcNS;
        const int j = it % ntiles;
        const bool pass_b = it >= ntiles;
        if (pass_b && it == ntiles) {  // combine the two halves' (m, l) once per item
          stat[(hf * 2 + 0) * 128 + i] = m;
          stat[(hf * 2 + 1) * 128 + i] = l;
          asm volatile("bar.sync 1, 256;" ::: "memory");
          const float mo = stat[((1 - hf) * 2 + 0) * 128 + i], lo = stat[((1 - hf) * 2 + 1) * 128 + i];
          const float mm = fmaxf(m, mo);
          const float ll = (mm == -INFINITY) ? 0.f : l * ex2_approx(m - mm) + lo * ex2_approx(mo - mm);
          mfin = ll > 0.f ? mm + __log2f(ll) : 0.f;
          l = ll;
        }
        const bool tree = j >= npt;
        const int lim = tree ? 0 : min(Pr - j * kTcNK - hf * 32, 32);  // visible prefix columns
        mbar_wait(&s_full[sb], (gs / kTcNS) & 1);
        tc_fence_after();
        uint32_t v[32];
#ifdef TA_TC_NOSOFTMAX
        tc_fence_before();
        mbar_arrive(&s_free[sb]);
        if (pass_b) {
          const int pbuf = pb & 1;
          if (pb >= 2) mbar_wait(&p_free[pbuf], ((pb >> 1) & 1) ^ 1);
          fence_proxy_async_smem();
          mbar_arrive(&p_full[pbuf]);
          ++pb;
        }
        continue;
#endif
        tmem_ld_32x32b_x32(trow + sb * kTcNK + hf * 32, v);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&s_free[sb]);
        float x[32];
        const bool full = a != 0ull && !tree && lim >= 32;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          bool ok;
          if (full) ok = true;
          else if (tree) ok = (ah >> e) & 1ull;
          else ok = a != 0ull && e < lim;
          x[e] = ok ? __uint_as_float(v[e]) : -INFINITY;
        }
        if (!pass_b) {
          float mr = -INFINITY;
#pragma unroll
          for (int e = 0; e < 32; ++e) mr = fmaxf(mr, x[e]);
          const float mx = fmaxf(m, mr * c2);
          if (mx != -INFINITY) {
            float s0 = 0.f, s1 = 0.f;
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              s0 += ex2_approx(fmaf(x[e], c2, -mx));
              s1 += ex2_approx(fmaf(x[e + 1], c2, -mx));
            }
            l = l * ex2_approx(m - mx) + (s0 + s1);
            m = mx;
          }
        } else {
          uint32_t w16[16];
#pragma unroll
          for (int h = 0; h < 16; ++h)
            w16[h] = pk_bf16(ex2_approx(fmaf(x[2 * h], c2, -mfin)), ex2_approx(fmaf(x[2 * h + 1], c2, -mfin)));
          const int pbuf = pb & 1;
          if (pb >= 2) mbar_wait(&p_free[pbuf], ((pb >> 1) & 1) ^ 1);
          const uint32_t rowb = aProw + pbuf * kTcPBuf;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t ch = static_cast<uint32_t>((hf * 4 + q) ^ (i & 7));
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowb + ch * 16), "r"(w16[4 * q]),
                         "r"(w16[4 * q + 1]), "r"(w16[4 * q + 2]), "r"(w16[4 * q + 3])
                         : "memory");
          }
          fence_proxy_async_smem();
          mbar_arrive(&p_full[pbuf]);
          ++pb;
        }
      }
      // epilogue: O (normalised already) -> bf16 global (this half's 64 columns), lse
      mbar_wait(o_done, wi & 1);
      tc_fence_after();
      uint32_t v[2][32];
      tmem_ld_32x32b_x32(trow + kTcNS * kTcNK + hf * 64, v[0]);
      tmem_ld_32x32b_x32(trow + kTcNS * kTcNK + hf * 64 + 32, v[1]);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(o_free);
      if (i < rows) {
        uint16_t* orow = p.Oout + (((size_t)r * N1 + s_row) * p.Hq + hk * G + g) * D + hf * 64;
        const bool live = a != 0ull;
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 o4;
            o4.x = live ? pk_bf16(__uint_as_float(v[c][8 * q + 0]), __uint_as_float(v[c][8 * q + 1])) : 0u;
            o4.y = live ? pk_bf16(__uint_as_float(v[c][8 * q + 2]), __uint_as_float(v[c][8 * q + 3])) : 0u;
            o4.z = live ? pk_bf16(__uint_as_float(v[c][8 * q + 4]), __uint_as_float(v[c][8 * q + 5])) : 0u;
            o4.w = live ? pk_bf16(__uint_as_float(v[c][8 * q + 6]), __uint_as_float(v[c][8 * q + 7])) : 0u;
            *reinterpret_cast<uint4*>(orow + c * 32 + q * 8) = o4;
          }
        if (hf == 0)
          p.lse_out[((size_t)r * N1 + s_row) * p.Hq + hk * G + g] = (live && l > 0.f) ? mfin * kLn2 : -INFINITY;
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");  // anc / stat are rewritten by the next item
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}


// ------------------------------------------------------------------------------ tcgen05 forward, one pass
// k_ta_fwd_tc2: one pass over the key tiles with an online softmax and lazy O rescaling, two
// work items in flight per SM.  The CTA holds two independent groups of 6 warps (group g = warps
// 6g .. 6g+5): a TMA producer (Q, then K and V tiles of 64 keys through two 2-stage rings), an MMA
// issuer (S = Q K^T into one of two 64-column TMEM buffers, O += P V into a 128-column TMEM
// accumulator) and 4 softmax warps (thread = query row = TMEM lane).  Per tile the softmax thread
// takes the row max; only when it exceeds the running max by more than 2^8 (log2 domain) does it
// rescale O in TMEM (wait for the previous P V, tcgen05.ld / scale / tcgen05.st) — otherwise P is
// computed against the stale max (values <= 256, exact in fp32, fine in bf16).  P goes to shared
// memory as the K-major A operand.  While one group runs its softmax, the tensor core works on the
// other group's S / P V, so the MMA <-> softmax round trips of the single-item kernel (k_ta_fwd_tc,
// two passes) overlap.  Work item = (request, KV head) with its G (N+1) <= 128 query rows.
constexpr int kT2NK = 64;
constexpr int kT2Slot = kT2NK * 128 * 2;            // 16 KB: K tile (2 K-major atoms) or V tile (2 MN slices)
// GRP work items per CTA (independent groups of 6 warps), KST / VST K / V ring stages, PB P
// buffers per group.  <2, 2, 2, 1>: two items in flight, 112 KB each; <1, 4, 4, 2>: one item
// with deep rings (192 KB: ~4 tiles of K and V in flight per SM)
template <int GRP, int KST, int VST, int PB>
struct TcPlan {
  static constexpr int kThreads = GRP * 192;
  static constexpr int kOffK = 32768;               // after Q (2 atoms of 128 rows x 128 B)
  static constexpr int kOffV = kOffK + KST * kT2Slot;
  static constexpr int kOffP = kOffV + VST * kT2Slot;
  static constexpr int kGrp = kOffP + PB * 128 * kT2NK * 2;
  static constexpr int kOffBar = GRP * kGrp;
  static constexpr size_t kSmem = kOffBar + 2048 + 1024;  // barriers + anc + TMEM holder + parents, alignment
  static_assert(kSmem <= 232448, "smem");
  static_assert(2 + 2 * KST + 2 * VST + 4 + 2 * PB + 3 <= 32, "barriers per group");
};

template <int GRP, int KST, int VST, int PB>
__global__ void __launch_bounds__(GRP * 192, 1) k_ta_fwd_tc2(const __grid_constant__ TaTcMaps maps, TaParams p) {
  using Plan = TcPlan<GRP, KST, VST, PB>;
  constexpr int kT2OffK = Plan::kOffK, kT2OffV = Plan::kOffV, kT2OffP = Plan::kOffP, kT2Grp = Plan::kGrp;
  constexpr int kT2OffBar = Plan::kOffBar;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = warp / 6, role = warp - grp * 6;
  uint8_t* gs = smem + grp * kT2Grp;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kT2OffBar);
  uint64_t* gb = bars + grp * 32;
  uint64_t* q_full = gb + 0;
  uint64_t* q_free = gb + 1;
  uint64_t* k_full = gb + 2;                 // [KST]
  uint64_t* k_empty = k_full + KST;          // [KST]
  uint64_t* v_full = k_empty + KST;          // [VST]
  uint64_t* v_empty = v_full + VST;          // [VST]
  uint64_t* s_full = v_empty + VST;          // [2]
  uint64_t* s_free = s_full + 2;             // [2]
  uint64_t* p_full = s_free + 2;             // [PB]
  uint64_t* p_free = p_full + PB;            // [PB]
  uint64_t* o_ready = p_free + PB;
  uint64_t* o_done = o_ready + 1;
  uint64_t* o_free = o_done + 1;
  uint64_t* anc = bars + 64 + grp * 40;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 160);
  int32_t* par_s = reinterpret_cast<int32_t*>(bars + 168 + grp * 16);  // the request's parents (N <= 32)
  const int G = p.G, N1 = p.N1;
  const int nwork = p.R * p.Hkv;
  {  // Q rows >= G (N+1) are never loaded: zero them once so their scores are 0 (unmasked, finite)
    const int rows = G * N1;
    for (int idx = threadIdx.x; idx < GRP * 2 * (128 - rows) * 8; idx += blockDim.x) {
      const int c = idx & 7, row = rows + (idx >> 3) % (128 - rows), part = (idx >> 3) / (128 - rows);
      *reinterpret_cast<uint4*>(smem + (part >> 1) * kT2Grp + (part & 1) * 16384 + row * 128 + c * 16) =
          make_uint4(0u, 0u, 0u, 0u);
    }
    fence_proxy_async_smem();
  }

  if (threadIdx.x == 0) {
    for (int g2 = 0; g2 < GRP; ++g2) {
      uint64_t* b = bars + g2 * 32;
      int o = 0;
      for (int k = 0; k < 2 + 2 * KST + 2 * VST + 2; ++k) mbar_init(&b[o++], 1);  // q, k, v rings, s_full
      for (int k = 0; k < 2; ++k) mbar_init(&b[o++], 128);                          // s_free
      for (int k = 0; k < PB; ++k) mbar_init(&b[o++], 128);                         // p_full
      for (int k = 0; k < PB; ++k) mbar_init(&b[o++], 1);                           // p_free
      mbar_init(&b[o++], 1);    // o_ready
      mbar_init(&b[o++], 1);    // o_done
      mbar_init(&b[o++], 128);  // o_free
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<GRP * 256>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder + grp * 256;  // S0 +0, S1 +64, O +128
  const int wstep = GRP * gridDim.x;

  if (role == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      if (grp == 0) {
        tma_prefetch_desc(&maps.Q);
        tma_prefetch_desc(&maps.Kp);
        tma_prefetch_desc(&maps.Vp);
        tma_prefetch_desc(&maps.Kt);
        tma_prefetch_desc(&maps.Vt);
      }
      uint32_t kc = 0, vc = 0;
      int wi = 0;
      for (int w = GRP * blockIdx.x + grp; w < nwork; w += wstep, ++wi) {
        const int r = w / p.Hkv, hk = w - r * p.Hkv;
        int p0, Pr;
        prefix_of(p, r, p0, Pr, hk == 0);
        const int npt = (Pr + kT2NK - 1) / kT2NK, nt = npt + 1;
        if (wi > 0) mbar_wait_sleep(q_free, (wi - 1) & 1);
        mbar_arrive_expect_tx(q_full, 2u * 128u * G * N1);
        tma_load_3d(&maps.Q, q_full, gs, 0, hk * G, r * N1);
        tma_load_3d(&maps.Q, q_full, gs + 16384, 64, hk * G, r * N1);
        for (int j = 0; j < nt; ++j) {
          const CUtensorMap* mk = j < npt ? &maps.Kp : &maps.Kt;
          const CUtensorMap* mv = j < npt ? &maps.Vp : &maps.Vt;
          const int z = j < npt ? p0 + j * kT2NK : r * N1;
          const uint32_t ks = kc % KST, vs = vc % VST;
          if (kc >= KST) mbar_wait_sleep(&k_empty[ks], ((kc / KST) & 1) ^ 1);
          mbar_arrive_expect_tx(&k_full[ks], kT2Slot);
          uint8_t* kd = gs + kT2OffK + ks * kT2Slot;
          tma_load_3d(mk, &k_full[ks], kd, 0, hk, z);
          tma_load_3d(mk, &k_full[ks], kd + kT2NK * 128, 64, hk, z);
          ++kc;
          if (vc >= VST) mbar_wait_sleep(&v_empty[vs], ((vc / VST) & 1) ^ 1);
          mbar_arrive_expect_tx(&v_full[vs], kT2Slot);
          uint8_t* vd = gs + kT2OffV + vs * kT2Slot;
          tma_load_3d(mv, &v_full[vs], vd, 0, hk, z);
          tma_load_3d(mv, &v_full[vs], vd + kT2NK * 128, 64, hk, z);
          ++vc;
        }
      }
    }
  } else if (role == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idS = umma_idesc_bf16(128, kT2NK, false, false);
      constexpr uint32_t idPV = umma_idesc_bf16(128, 128, false, true);
      const uint32_t aQ = smem_u32(gs), aP = smem_u32(gs + kT2OffP);
      uint32_t kc = 0, vc = 0, sc = 0, pc = 0;
      int wi = 0;
      auto pv_issue = [&](int jj) {
        const uint32_t vs = vc % VST, pbuf = pc % PB;
        mbar_wait(&v_full[vs], (vc / VST) & 1);
        mbar_wait(&p_full[pbuf], (pc / PB) & 1);
        if (jj == 0 && wi > 0) mbar_wait(o_free, (wi - 1) & 1);  // the epilogue read the previous O
        tc_fence_after();
        const uint32_t vb = smem_u32(gs + kT2OffV + vs * kT2Slot);
#pragma unroll
        for (int kk = 0; kk < kT2NK / 16; ++kk)
          umma_bf16(tmem + 128, kmaj_desc(aP + pbuf * (128 * kT2NK * 2), kk, 128), mnmaj_desc(vb, kk, kT2NK), idPV,
                    (jj > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&p_free[pbuf]);
        umma_commit(&v_empty[vs]);
        umma_commit(o_ready);
        ++vc;
        ++pc;
      };
      for (int w = GRP * blockIdx.x + grp; w < nwork; w += wstep, ++wi) {
        const int r = w / p.Hkv;
        int p0, Pr;
        prefix_of(p, r, p0, Pr, false);
        const int nt = (Pr + kT2NK - 1) / kT2NK + 1;
        mbar_wait(q_full, wi & 1);
        for (int j = 0; j < nt; ++j) {
          const uint32_t ks = kc % KST, sb = sc & 1;
          mbar_wait(&k_full[ks], (kc / KST) & 1);
          if (sc >= 2) mbar_wait(&s_free[sb], ((sc >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t kb = smem_u32(gs + kT2OffK + ks * kT2Slot);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16(tmem + sb * kT2NK, kmaj_desc(aQ, kk, 128), kmaj_desc(kb, kk, kT2NK), idS, kk > 0);
          umma_commit(&s_full[sb]);
          umma_commit(&k_empty[ks]);
          ++kc;
          ++sc;
          if (j == nt - 1) umma_commit(q_free);
          if (j >= 1) pv_issue(j - 1);
        }
        pv_issue(nt - 1);
        umma_commit(o_done);
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax (4 warps, thread = row)
    const int q4 = warp & 3;
    const int i = q4 * 32 + lane;
    const int rows = G * N1;
    const uint32_t trow = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
    const uint32_t aProw = smem_u32(gs + kT2OffP) + i * 128;
    const float c2 = p.c2;
    const int st_id = (role - 2) * 32 + lane;  // 0..127
    uint32_t sc = 0, pvc = 0;
    int wi = 0;
    for (int w = GRP * blockIdx.x + grp; w < nwork; w += wstep, ++wi) {
      const int r = w / p.Hkv, hk = w - r * p.Hkv;
      int p0, Pr;
      prefix_of(p, r, p0, Pr, false);
      const int npt = (Pr + kT2NK - 1) / kT2NK, nt = npt + 1;
      {  // ancestor masks of this request (bit t = tree key t visible): the parents are loaded in
         // parallel into shared memory, then each row walks its ancestor chain there
        const int nn = p.num_nodes ? p.num_nodes[r] : p.N;
        if (st_id < p.N) par_s[st_id] = p.parents ? p.parents[(size_t)r * p.N + st_id] : st_id - 1;
        asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");
        if (st_id < N1) {
          const int s = st_id;
          bool bad = nn < 0 || nn > p.N;
          uint64_t m = 0;
          if (!bad) {
            if (s == 0) {
              m = 1ull;
            } else if (s - 1 < nn) {
              int cur = s - 1;
              m = 1ull | (1ull << s);
              for (int k = 0; k <= p.N; ++k) {
                const int par = par_s[cur];
                if (par < -1 || par >= cur) { bad = true; break; }
                if (par < 0) break;
                m |= 1ull << (par + 1);
                cur = par;
              }
            }
          }
          if (bad && p.status && hk == 0) atomicOr(p.status, (uint32_t)AURORA_STATUS_STRUCTURE);
          anc[s] = bad ? 0ull : m;
        }
      }
      asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");
      const int s_row = i / G, g = i - s_row * G;
      const uint64_t a = i < rows ? anc[s_row] : 0ull;
      // Rows that are not output (a = 0: padding rows, whose Q rows are zero in shared memory, and
      // invalid tree rows, written as O = 0, lse = -inf) need no mask: their scores are finite.
      // So a prefix tile with every key inside the prefix is unmasked for the whole warp (the
      // common case); the request's last prefix tile and its tree tile take the masked path.
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < nt; ++j, ++sc) {
        const uint32_t sb = sc & 1;
        const bool tree = j == npt;
        const int lim = tree ? 0 : Pr - j * kT2NK;
        uint64_t vis = tree ? a : (lim >= kT2NK ? ~0ull : ((1ull << max(lim, 0)) - 1ull));
        if (a == 0ull) vis = ~0ull;
        const bool wfull = __all_sync(0xffffffffu, vis == ~0ull);
        mbar_wait(&s_full[sb], (sc >> 1) & 1);
        tc_fence_after();
        float x[64];
        tmem_ld_32x32b_x32(trow + sb * kT2NK, reinterpret_cast<uint32_t(&)[32]>(x[0]));
        tmem_ld_32x32b_x32(trow + sb * kT2NK + 32, reinterpret_cast<uint32_t(&)[32]>(x[32]));
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&s_free[sb]);
        if (!wfull) {
          const uint32_t vlo = static_cast<uint32_t>(vis), vhi = static_cast<uint32_t>(vis >> 32);
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            x[e] = ((vlo >> e) & 1u) ? x[e] : -INFINITY;
            x[e + 32] = ((vhi >> e) & 1u) ? x[e + 32] : -INFINITY;
          }
        }
        // row max: a tree of independent max3 (no 64-long dependency chain)
        float t21[22];
#pragma unroll
        for (int q = 0; q < 21; ++q) t21[q] = fmaxf(fmaxf(x[3 * q], x[3 * q + 1]), x[3 * q + 2]);
        t21[21] = x[63];
        float t7[8];
#pragma unroll
        for (int q = 0; q < 7; ++q) t7[q] = fmaxf(fmaxf(t21[3 * q], t21[3 * q + 1]), t21[3 * q + 2]);
        t7[7] = t21[21];
        float mt = fmaxf(fmaxf(fmaxf(t7[0], t7[1]), fmaxf(t7[2], t7[3])), fmaxf(fmaxf(t7[4], t7[5]), fmaxf(t7[6], t7[7])));
        mt *= c2;
        // lazy rescale: only when a row's max grew by more than 2^8 (log2 domain); the TMEM
        // load / store are warp-collective, so the warp rescales together (factor 1 on the
        // rows that keep their max)
        const bool grow = mt > m + 8.f;
        const bool resc = grow && m != -INFINITY;
        const float f = resc ? ex2_approx(m - mt) : 1.f;
        if (resc) l *= f;
        if (__any_sync(0xffffffffu, resc)) {
          mbar_wait(o_ready, (pvc - 1) & 1);  // the previous P V (the last one) has landed
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(trow + 128 + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * f);
            tmem_st_32x32b_x32(trow + 128 + c * 32, o);
          }
          tmem_st_wait();
        }
        if (grow) m = mt;
        uint32_t w32[32];
        float sacc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const float nm = m == -INFINITY ? 0.f : -m;  // rows with no visible key yet: e = 0, not NaN
#pragma unroll
        for (int h = 0; h < 32; ++h) {
          const float e0 = ex2_approx(fmaf(x[2 * h], c2, nm)), e1 = ex2_approx(fmaf(x[2 * h + 1], c2, nm));
          sacc[(2 * h) & 7] += e0;
          sacc[(2 * h + 1) & 7] += e1;
          w32[h] = pk_bf16(e0, e1);
        }
        l += ((sacc[0] + sacc[1]) + (sacc[2] + sacc[3])) + ((sacc[4] + sacc[5]) + (sacc[6] + sacc[7]));
        const uint32_t pbuf = pvc % PB;
        if (pvc >= PB) mbar_wait(&p_free[pbuf], ((pvc / PB) & 1) ^ 1);  // the P V that last read this buffer
        const uint32_t prow = aProw + pbuf * (128 * kT2NK * 2);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint32_t ch = static_cast<uint32_t>(c ^ (i & 7));
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(prow + ch * 16), "r"(w32[4 * c]),
                       "r"(w32[4 * c + 1]), "r"(w32[4 * c + 2]), "r"(w32[4 * c + 3])
                       : "memory");
        }
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&p_full[pbuf]);
        ++pvc;
      }
      // epilogue: O / l -> bf16 global, lse
      mbar_wait(o_done, wi & 1);
      tc_fence_after();
      uint32_t o[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(trow + 128 + c * 32, o[c]);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(o_free);
      if (i < rows) {
        const bool live = a != 0ull && l > 0.f;
        const float inv = live ? 1.f / l : 0.f;
        uint16_t* orow = p.Oout + (((size_t)r * N1 + s_row) * p.Hq + hk * G + g) * D;
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 o4;
            o4.x = pk_bf16(__uint_as_float(o[c][8 * q + 0]) * inv, __uint_as_float(o[c][8 * q + 1]) * inv);
            o4.y = pk_bf16(__uint_as_float(o[c][8 * q + 2]) * inv, __uint_as_float(o[c][8 * q + 3]) * inv);
            o4.z = pk_bf16(__uint_as_float(o[c][8 * q + 4]) * inv, __uint_as_float(o[c][8 * q + 5]) * inv);
            o4.w = pk_bf16(__uint_as_float(o[c][8 * q + 6]) * inv, __uint_as_float(o[c][8 * q + 7]) * inv);
            *reinterpret_cast<uint4*>(orow + c * 32 + q * 8) = o4;
          }
        p.lse_out[((size_t)r * N1 + s_row) * p.Hq + hk * G + g] = live ? (m + __log2f(l)) * kLn2 : -INFINITY;
      }
      asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");  // anc is rewritten by the next item
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<GRP * 256>(*tmem_holder);
  }
}

// ------------------------------------------------------------------------------ tcgen05 backward
// k_ta_bwd_tc: the one-kernel backward on the tensor cores.  Work item = (request, KV head) with
// all its G (N+1) <= 128 query rows (so every key's dK / dV is complete after one tile step: no
// atomics), one item per CTA and SM, key tiles of 64.  Per tile j the MMA warp issues
//   S = Q K^T and dP = dO V^T                       (M 128 rows, N 64 keys, K 128 dh)  -> TMEM
// and, once the compute warps wrote P and dS = scale P (dP - D) (bf16, shared memory):
//   dV^T = dO^T P, dK^T = Q^T dS                    (M 128 dh, N 64 keys, K 128 rows)  -> TMEM
//   dQ += dS K                                      (M 128 rows, N 128 dh, K 64 keys)  -> TMEM
// every operand read straight from the swizzled tiles TMA loaded: Q / dO serve as K-major A
// (rows x dh) and as MN-major A (dh x rows); the K tile as K-major B (keys x dh) and MN-major B
// (dh x keys); P / dS as K-major A and MN-major B.  The 4 compute warps (thread = row for the
// softmax, = dh lane for the dK / dV epilogue) overlap the next tile's softmax with the
// gradient MMAs of the previous one (S, dP and P / dS double-buffered).
// TMEM columns: S[2] 0 / 64, dP[2] 128 / 192, dQ 256..383, dV^T 384..447, dK^T 448..511.
struct TaBwdMaps {
  CUtensorMap Q, dO, Kp, Vp, Kt, Vt;
};
constexpr int kTbKST = 4, kTbVST = 2;              // K / V ring depths (a K slot is held until the
                                                   // tile's dQ MMA, a V slot only until its dP MMA)
constexpr int kTbOffQ = 0, kTbOffDO = 32768, kTbOffK = 65536;
constexpr int kTbOffV = kTbOffK + kTbKST * kT2Slot;
constexpr int kTbOffP = kTbOffV + kTbVST * kT2Slot;  // 2 x [128 rows x 64 keys] bf16
constexpr int kTbOffDS = kTbOffP + 2 * 16384;
constexpr int kTbOffBar = kTbOffDS + 2 * 16384;    // 224 KB
constexpr size_t kSmemTb = kTbOffBar + 1024 + 1024;

#ifndef TA_BWD_KV_KSTEPS
#define TA_BWD_KV_KSTEPS 8  // (experiments only: fewer K steps in the dV^T / dK^T MMAs)
#endif
#ifndef TA_BWD_DP_KSTEPS
#define TA_BWD_DP_KSTEPS 8  // (experiments only: fewer K steps in the dP MMAs)
#endif
#ifndef TA_BWD_CW
#define TA_BWD_CW 16
#endif
constexpr int kTbCW = TA_BWD_CW;                    // compute warps (8 or 16: 2 or 4 per TMEM lane quadrant)
constexpr int kTbCompute = 32 * kTbCW;             // compute threads
constexpr int kTbSplit = kTbCW / 4;                // warps per lane quadrant
constexpr int kTbCols = 64 / kTbSplit;             // key columns of S / dP / dV^T / dK^T per warp
constexpr int kTbQCols = 128 / kTbSplit;           // dQ columns per warp
static_assert(kTbCW == 8 || kTbCW == 16, "compute warps");
template <int N>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[N]) {
  if constexpr (N == 32) tmem_ld_32x32b_x32(taddr, r);
  else tmem_ld_32x32b_x16(taddr, r);
}
__global__ void __launch_bounds__(64 + kTbCompute, 1) k_ta_bwd_tc(const __grid_constant__ TaBwdMaps maps, TaParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTbOffBar);
  uint64_t* q_full = bars + 0;
  uint64_t* q_free = bars + 1;
  uint64_t* k_full = bars + 2;               // [kTbKST]
  uint64_t* k_empty = k_full + kTbKST;       // [kTbKST]
  uint64_t* v_full = k_empty + kTbKST;       // [kTbVST]
  uint64_t* v_empty = v_full + kTbVST;       // [kTbVST]
  uint64_t* s_full = bars + 14;   // [2] S and dP of a tile in TMEM
  uint64_t* s_free = bars + 16;   // [2]
  uint64_t* pd_full = bars + 18;  // [2] P and dS of a tile in smem
  uint64_t* pd_free = bars + 20;  // [2]
  uint64_t* kv_full = bars + 22;  // dV^T, dK^T of a tile in TMEM
  uint64_t* kv_free = bars + 23;
  uint64_t* dq_done = bars + 24;
  uint64_t* dq_free = bars + 25;
  static_assert(2 * kTbKST + 2 * kTbVST == 12, "barrier layout: s_full starts at 14");
  uint64_t* anc = bars + 32;      // [40]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 80);
  int32_t* par_s = reinterpret_cast<int32_t*>(bars + 88);  // the request's parents (N <= 32)
  const int G = p.G, N1 = p.N1;
  const int nwork = p.R * p.Hkv;
  if (threadIdx.x == 0) {
    for (int k = 0; k < 16; ++k) mbar_init(&bars[k], 1);            // q, k / v rings, s_full
    for (int k = 16; k < 18; ++k) mbar_init(&bars[k], kTbCompute);  // s_free
    for (int k = 18; k < 20; ++k) mbar_init(&bars[k], kTbCompute);  // pd_full
    for (int k = 20; k < 22; ++k) mbar_init(&bars[k], 1);           // pd_free
    mbar_init(kv_full, 1);
    mbar_init(kv_free, kTbCompute);
    mbar_init(dq_done, 1);
    mbar_init(dq_free, kTbCompute);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_holder);
  {  // rows >= G (N+1) of the Q / dO tiles are never loaded but feed the dV^T / dK^T sums over
     // rows (times P = dS = 0): zero them once so stale shared memory cannot inject NaN
    const int rows = G * N1;
    for (int idx = threadIdx.x; idx < (128 - rows) * 4 * 8; idx += blockDim.x) {
      const int row = rows + idx / 32, part = (idx / 8) & 3, c = idx & 7;
      const int off = (part >> 1) * kTbOffDO + (part & 1) * 16384 + row * 128 + c * 16;
      *reinterpret_cast<uint4*>(smem + off) = make_uint4(0u, 0u, 0u, 0u);
    }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&maps.Q);
      tma_prefetch_desc(&maps.dO);
      tma_prefetch_desc(&maps.Kp);
      tma_prefetch_desc(&maps.Vp);
      tma_prefetch_desc(&maps.Kt);
      tma_prefetch_desc(&maps.Vt);
      uint32_t kc = 0, vc = 0;
      int wi = 0;
      for (int w = blockIdx.x; w < nwork; w += gridDim.x, ++wi) {
        const int r = w / p.Hkv, hk = w - r * p.Hkv;
        int p0, Pr;
        prefix_of(p, r, p0, Pr, false);
        const int npt = (Pr + kT2NK - 1) / kT2NK, nt = npt + 1;
        if (wi > 0) mbar_wait_sleep(q_free, (wi - 1) & 1);
        mbar_arrive_expect_tx(q_full, 4u * 128u * G * N1);
        tma_load_3d(&maps.Q, q_full, smem + kTbOffQ, 0, hk * G, r * N1);
        tma_load_3d(&maps.Q, q_full, smem + kTbOffQ + 16384, 64, hk * G, r * N1);
        tma_load_3d(&maps.dO, q_full, smem + kTbOffDO, 0, hk * G, r * N1);
        tma_load_3d(&maps.dO, q_full, smem + kTbOffDO + 16384, 64, hk * G, r * N1);
        for (int j = 0; j < nt; ++j) {
          const CUtensorMap* mk = j < npt ? &maps.Kp : &maps.Kt;
          const CUtensorMap* mv = j < npt ? &maps.Vp : &maps.Vt;
          const int z = j < npt ? p0 + j * kT2NK : r * N1;
          const uint32_t ks = kc % kTbKST, vs = vc % kTbVST;
          if (kc >= kTbKST) mbar_wait_sleep(&k_empty[ks], ((kc / kTbKST) & 1) ^ 1);
          mbar_arrive_expect_tx(&k_full[ks], kT2Slot);
          uint8_t* kd = smem + kTbOffK + ks * kT2Slot;
          tma_load_3d(mk, &k_full[ks], kd, 0, hk, z);
          tma_load_3d(mk, &k_full[ks], kd + kT2NK * 128, 64, hk, z);
          ++kc;
          if (vc >= kTbVST) mbar_wait_sleep(&v_empty[vs], ((vc / kTbVST) & 1) ^ 1);
          mbar_arrive_expect_tx(&v_full[vs], kT2Slot);
          uint8_t* vd = smem + kTbOffV + vs * kT2Slot;
          tma_load_3d(mv, &v_full[vs], vd, 0, hk, z);
          tma_load_3d(mv, &v_full[vs], vd + kT2NK * 128, 64, hk, z);
          ++vc;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idS = umma_idesc_bf16(128, kT2NK, false, false);     // S, dP
      constexpr uint32_t idT = umma_idesc_bf16(128, kT2NK, true, true);       // dV^T, dK^T
      constexpr uint32_t idQ = umma_idesc_bf16(128, 128, false, true);        // dQ
      const uint32_t aQ = smem_u32(smem + kTbOffQ), aDO = smem_u32(smem + kTbOffDO);
      uint32_t kc = 0, vc = 0, sc = 0, gc = 0;  // K / V loads consumed, S tiles issued, gradient steps issued
      int wi = 0;
      for (int w = blockIdx.x; w < nwork; w += gridDim.x, ++wi) {
        const int r = w / p.Hkv;
        int p0, Pr;
        prefix_of(p, r, p0, Pr, false);
        const int nt = (Pr + kT2NK - 1) / kT2NK + 1;
        mbar_wait(q_full, wi & 1);
        uint32_t kslot_prev = 0;
        auto grad = [&](int jj, uint32_t kslot) {  // gradient MMAs of tile jj (P / dS written)
          const uint32_t pb = gc & 1;
          mbar_wait(&pd_full[pb], (gc >> 1) & 1);
          if (gc >= 1) mbar_wait(kv_free, (gc - 1) & 1);            // the epilogue read dV^T / dK^T
          if (jj == 0 && wi > 0) mbar_wait(dq_free, (wi - 1) & 1);  // the epilogue read the last dQ
          tc_fence_after();
          const uint32_t aP = smem_u32(smem + kTbOffP + pb * 16384), aS = smem_u32(smem + kTbOffDS + pb * 16384);
          const uint32_t kb = smem_u32(smem + kTbOffK + kslot * kT2Slot);
#pragma unroll
          for (int kk = 0; kk < TA_BWD_KV_KSTEPS; ++kk)  // K = 128 rows
            umma_bf16(tmem + 384, mnmaj_desc(aDO, kk, 128), mnmaj_desc(aP, kk, 128), idT, kk > 0);
#pragma unroll
          for (int kk = 0; kk < TA_BWD_KV_KSTEPS; ++kk)
            umma_bf16(tmem + 448, mnmaj_desc(aQ, kk, 128), mnmaj_desc(aS, kk, 128), idT, kk > 0);
#pragma unroll
          for (int kk = 0; kk < kT2NK / 16; ++kk)  // K = 64 keys
            umma_bf16(tmem + 256, kmaj_desc(aS, kk, 128), mnmaj_desc(kb, kk, kT2NK), idQ, (jj > 0 || kk > 0) ? 1u : 0u);
          umma_commit(kv_full);
          umma_commit(&pd_free[pb]);
          umma_commit(&k_empty[kslot]);  // K: S and dQ done
          ++gc;
        };
        for (int j = 0; j < nt; ++j) {
          const uint32_t ks = kc % kTbKST, vs = vc % kTbVST, sb = sc & 1;
          mbar_wait(&k_full[ks], (kc / kTbKST) & 1);
          mbar_wait(&v_full[vs], (vc / kTbVST) & 1);
          if (sc >= 2) mbar_wait(&s_free[sb], ((sc >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t kb = smem_u32(smem + kTbOffK + ks * kT2Slot), vb = smem_u32(smem + kTbOffV + vs * kT2Slot);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16(tmem + sb * kT2NK, kmaj_desc(aQ, kk, 128), kmaj_desc(kb, kk, kT2NK), idS, kk > 0);
#pragma unroll
          for (int kk = 0; kk < TA_BWD_DP_KSTEPS; ++kk)
            umma_bf16(tmem + 128 + sb * kT2NK, kmaj_desc(aDO, kk, 128), kmaj_desc(vb, kk, kT2NK), idS, kk > 0);
          umma_commit(&s_full[sb]);
          umma_commit(&v_empty[vs]);  // V: dP done
          ++vc;
          ++sc;
          if (j >= 1) grad(j - 1, kslot_prev);
          kslot_prev = ks;
          ++kc;
        }
        grad(nt - 1, kslot_prev);
        umma_commit(dq_done);
        umma_commit(q_free);
      }
    }
  } else {
    // ---------------------------------------------------------------- compute (kTbCW warps)
    // kTbSplit warps per TMEM lane quadrant: warp slice hf owns key columns [kTbCols hf, +kTbCols)
    // of S / dP and of dV^T / dK^T, and dQ columns [kTbQCols hf, +kTbQCols)
    const int q4 = warp & 3;
    const int hf = (warp - 2) >> 2;
    const int i = q4 * 32 + lane;  // row (softmax) or dh lane (dK / dV epilogue)
    const int rows = G * N1;
    const uint32_t trow = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
    const float c2 = p.c2, scale = p.scale;
    const int st_id = (warp - 2) * 32 + lane;  // 0 .. 255
    uint32_t sc = 0, gc = 0;
    int wi = 0;
    for (int w = blockIdx.x; w < nwork; w += gridDim.x, ++wi) {
      const int r = w / p.Hkv, hk = w - r * p.Hkv;
      int p0, Pr;
      prefix_of(p, r, p0, Pr, false);
      const int npt = (Pr + kT2NK - 1) / kT2NK, nt = npt + 1;
      const int s_row = i / G, g = i - s_row * G;
      const size_t rix = ((size_t)r * N1 + s_row) * p.Hq + hk * G + g;
      // this row's lse and its slice of O, loaded before the ancestor walk so their latency
      // overlaps it; D = rowsum(dO * O) is formed here from the dO tile the TMA brought in (no
      // separate pass over O and dO)
      const float lse_raw = i < rows ? p.lse[rix] : 0.f;
      uint4 o_sl[kTbQCols / 8];
#pragma unroll
      for (int c = 0; c < kTbQCols / 8; ++c)
        o_sl[c] = i < rows ? *reinterpret_cast<const uint4*>(p.O + rix * D + hf * kTbQCols + c * 8)
                           : make_uint4(0u, 0u, 0u, 0u);
      {  // ancestor masks: parents loaded in parallel into shared memory, walked there
        if (st_id < p.N) par_s[st_id] = p.parents ? p.parents[(size_t)r * p.N + st_id] : st_id - 1;
        asm volatile("bar.sync 1, %0;" ::"n"(kTbCompute) : "memory");
        if (st_id < N1) {
          const int s = st_id;
          const int nn = p.num_nodes ? p.num_nodes[r] : p.N;
          bool bad = nn < 0 || nn > p.N;
          uint64_t m = 0;
          if (!bad) {
            if (s == 0) {
              m = 1ull;
            } else if (s - 1 < nn) {
              int cur = s - 1;
              m = 1ull | (1ull << s);
              for (int k = 0; k <= p.N; ++k) {
                const int par = par_s[cur];
                if (par < -1 || par >= cur) { bad = true; break; }
                if (par < 0) break;
                m |= 1ull << (par + 1);
                cur = par;
              }
            }
          }
          anc[s] = bad ? 0ull : m;
        }
      }
      // D: this warp's kTbQCols columns of dO (row i of the swizzled K-major tile) times O, the
      // kTbSplit partials summed in slice order through the free P buffer (deterministic)
      mbar_wait(q_full, wi & 1);
      {
        float part = 0.f;
        const uint32_t arow = smem_u32(smem + kTbOffDO) + (hf * kTbQCols / 64) * 16384 + i * 128;
#pragma unroll
        for (int c = 0; c < kTbQCols / 8; ++c) {
          const uint32_t ch = static_cast<uint32_t>(((hf * kTbQCols % 64) / 8 + c) ^ (i & 7));
          const float4 dv4 = lds128(arow + ch * 16);
          const uint32_t dw4[4] = {__float_as_uint(dv4.x), __float_as_uint(dv4.y), __float_as_uint(dv4.z),
                                   __float_as_uint(dv4.w)};
          const uint32_t ow4[4] = {o_sl[c].x, o_sl[c].y, o_sl[c].z, o_sl[c].w};
#pragma unroll
          for (int q = 0; q < 4; ++q)
            part = fmaf(bf16_hi(dw4[q]), bf16_hi(ow4[q]), fmaf(bf16_lo(dw4[q]), bf16_lo(ow4[q]), part));
        }
        reinterpret_cast<float*>(smem + kTbOffP + (sc & 1) * 16384)[hf * 128 + i] = part;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kTbCompute) : "memory");
      float D_row = 0.f;
#pragma unroll
      for (int h2 = 0; h2 < kTbSplit; ++h2) D_row += reinterpret_cast<const float*>(smem + kTbOffP + (sc & 1) * 16384)[h2 * 128 + i];
      asm volatile("bar.sync 1, %0;" ::"n"(kTbCompute) : "memory");  // the buffer takes P / dS next
      const uint64_t a = i < rows ? anc[s_row] : 0ull;
      const float lse2 = (a != 0ull) ? lse_raw * kLog2e : 0.f;
      const float Di = (a != 0ull) ? D_row : 0.f;
      auto epilogue = [&](int jj) {  // dV^T / dK^T of tile jj -> global (thread = dh lane i)
        mbar_wait(kv_full, gc & 1);
        tc_fence_after();
        uint32_t dv[kTbCols], dk[kTbCols];
        tmem_ld_cols(trow + 384 + hf * kTbCols, dv);
        tmem_ld_cols(trow + 448 + hf * kTbCols, dk);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(kv_free);
        ++gc;
        const bool tree = jj == npt;
        const int nkeys = tree ? N1 : min(kT2NK, Pr - jj * kT2NK);
        uint16_t* gdv = tree ? p.dVt : p.dVp;
        uint16_t* gdk = tree ? p.dKt : p.dKp;
        const int64_t key0 = tree ? (int64_t)r * N1 : (int64_t)p0 + jj * kT2NK;
        // transpose through the P / dS buffer of tile jj (free: kv_full covers every MMA that read
        // it): [key][dh] bf16 rows of 256 B, then 16 B coalesced stores of whole key rows
        const uint32_t b = (sc - 1) & 1;
        const uint32_t sdv = smem_u32(smem + kTbOffP) + b * 16384, sdk = smem_u32(smem + kTbOffDS) + b * 16384;
        const uint32_t adv = sdv + (hf * kTbCols) * 256 + i * 2, adk = sdk + (hf * kTbCols) * 256 + i * 2;
#pragma unroll
        for (int t = 0; t < kTbCols; ++t) {  // unrolled: register-indexed dv / dk
          const uint16_t hv = __bfloat16_as_ushort(__float2bfloat16_rn(__uint_as_float(dv[t])));
          const uint16_t hk2 = __bfloat16_as_ushort(__float2bfloat16_rn(__uint_as_float(dk[t])));
          asm volatile("st.shared.b16 [%0], %1;" ::"r"(adv + t * 256), "h"(hv) : "memory");
          asm volatile("st.shared.b16 [%0], %1;" ::"r"(adk + t * 256), "h"(hk2) : "memory");
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kTbCompute) : "memory");
        const int part = st_id & 15;
#pragma unroll
        for (int u = 0; u < kT2NK * 16 / kTbCompute; ++u) {
          const int t = (st_id >> 4) + (kTbCompute / 16) * u;
          if (t < nkeys) {
            const int64_t o = ((key0 + t) * p.Hkv + hk) * D + part * 8;
            uint4 v4, k4;
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v4.x), "=r"(v4.y), "=r"(v4.z), "=r"(v4.w)
                         : "r"(sdv + t * 256 + part * 16));
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(k4.x), "=r"(k4.y), "=r"(k4.z), "=r"(k4.w)
                         : "r"(sdk + t * 256 + part * 16));
#ifndef TA_BWD_NO_KV_STORE
            *reinterpret_cast<uint4*>(gdv + o) = v4;
            *reinterpret_cast<uint4*>(gdk + o) = k4;
#else
            if ((v4.x ^ k4.y) == 0x12345678u) gdv[o] = 0;  // experiments only: keep the loads alive
#endif
          }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kTbCompute) : "memory");  // the buffer takes the next P / dS
      };
      for (int j = 0; j < nt; ++j, ++sc) {
        const uint32_t sb = sc & 1;
        const bool tree = j == npt;
        const int lim = tree ? 0 : Pr - j * kT2NK;
        mbar_wait(&s_full[sb], (sc >> 1) & 1);
        tc_fence_after();
        float x[kTbCols], dpv[kTbCols];
        tmem_ld_cols(trow + sb * kT2NK + hf * kTbCols, reinterpret_cast<uint32_t(&)[kTbCols]>(x));
        tmem_ld_cols(trow + 128 + sb * kT2NK + hf * kTbCols, reinterpret_cast<uint32_t(&)[kTbCols]>(dpv));
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&s_free[sb]);
        // visibility of this tile's keys; rows >= G (N+1) have zero Q / dO rows in shared memory
        // (P = 1, dP = 0, D = 0: they add nothing), so only real rows are masked, and a prefix tile
        // wholly inside the prefix needs no mask at all (warp-uniform fast path)
        uint64_t vis = tree ? a : (a == 0ull ? 0ull : (lim >= kT2NK ? ~0ull : ((1ull << max(lim, 0)) - 1ull)));
        if (i >= rows) vis = ~0ull;
        constexpr uint32_t kFullMask = kTbCols == 32 ? 0xFFFFFFFFu : ((1u << kTbCols) - 1u);
        const uint32_t vv = static_cast<uint32_t>(vis >> (hf * kTbCols)) & kFullMask;
        const bool wfull = __all_sync(0xffffffffu, vv == kFullMask);
        uint32_t pw[kTbCols / 2], dw[kTbCols / 2];
        const float nl = -lse2;
        const float sDi = -scale * Di;  // dS = P (scale dP - scale D)
        if (wfull) {
#pragma unroll
          for (int h = 0; h < kTbCols / 2; ++h) {
            const float e0 = ex2_approx(fmaf(x[2 * h], c2, nl)), e1 = ex2_approx(fmaf(x[2 * h + 1], c2, nl));
            pw[h] = pk_bf16(e0, e1);
            dw[h] = pk_bf16(e0 * fmaf(dpv[2 * h], scale, sDi), e1 * fmaf(dpv[2 * h + 1], scale, sDi));
          }
        } else {
#pragma unroll
          for (int h = 0; h < kTbCols / 2; ++h) {
            const bool ok0 = (vv >> (2 * h)) & 1u, ok1 = (vv >> (2 * h + 1)) & 1u;
            const float e0 = ok0 ? ex2_approx(fmaf(x[2 * h], c2, nl)) : 0.f;
            const float e1 = ok1 ? ex2_approx(fmaf(x[2 * h + 1], c2, nl)) : 0.f;
            // never 0 * NaN from masked keys
            const float d0 = ok0 ? scale * e0 * (dpv[2 * h] - Di) : 0.f;
            const float d1 = ok1 ? scale * e1 * (dpv[2 * h + 1] - Di) : 0.f;
            pw[h] = pk_bf16(e0, e1);
            dw[h] = pk_bf16(d0, d1);
          }
        }
        const uint32_t pb = (sc) & 1;
        if (sc >= 2) mbar_wait(&pd_free[pb], ((sc >> 1) & 1) ^ 1);
        const uint32_t prow = smem_u32(smem + kTbOffP + pb * 16384) + i * 128;
        const uint32_t drow = smem_u32(smem + kTbOffDS + pb * 16384) + i * 128;
#pragma unroll
        for (int cc = 0; cc < kTbCols / 8; ++cc) {
          const uint32_t ch = static_cast<uint32_t>((hf * (kTbCols / 8) + cc) ^ (i & 7));
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(prow + ch * 16), "r"(pw[4 * cc]),
                       "r"(pw[4 * cc + 1]), "r"(pw[4 * cc + 2]), "r"(pw[4 * cc + 3])
                       : "memory");
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(drow + ch * 16), "r"(dw[4 * cc]),
                       "r"(dw[4 * cc + 1]), "r"(dw[4 * cc + 2]), "r"(dw[4 * cc + 3])
                       : "memory");
        }
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&pd_full[pb]);
        if (j >= 1) epilogue(j - 1);
      }
      epilogue(nt - 1);
      // dQ (thread = row, this warp's 64 of the 128 columns): fp32 [row][dh]
      mbar_wait(dq_done, wi & 1);
      tc_fence_after();
      uint32_t dq[kTbQCols / 32][32];
#pragma unroll
      for (int c = 0; c < kTbQCols / 32; ++c) tmem_ld_32x32b_x32(trow + 256 + hf * kTbQCols + c * 32, dq[c]);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(dq_free);
      if (i < rows) {
        float* out = p.dQ + rix * D + hf * kTbQCols;
        const bool live = a != 0ull;
#pragma unroll
        for (int c = 0; c < kTbQCols / 32; ++c)
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *reinterpret_cast<float4*>(out + c * 32 + q * 4) =
                live ? make_float4(__uint_as_float(dq[c][4 * q]), __uint_as_float(dq[c][4 * q + 1]),
                                   __uint_as_float(dq[c][4 * q + 2]), __uint_as_float(dq[c][4 * q + 3]))
                     : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kTbCompute) : "memory");  // anc is rewritten by the next item
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ------------------------------------------------------------------------------ tree RoPE
// Block per tree row (request r, row s): position P_r + depth(s) (F4-R6; siblings share it),
// cos/sin of pos * theta^(-2i/dh) for the dh/2 frequencies computed once in double into shared
// memory, then every query head of the row (and every KV head of its tree key) is rotated in
// place (rotate-half pairs (i, i + dh/2)); inverse = the transposed rotation (for gradients).
template <typename TQ, typename TK>
__global__ void __launch_bounds__(128) k_ta_rope(TaParams p, TQ* __restrict__ Q, TK* __restrict__ Kt, int dh,
                                                 double log2_theta, int inverse) {
  __shared__ float s_cos[128], s_sin[128];
  __shared__ int s_pos;
  const int row = blockIdx.x, r = row / p.N1, s = row - r * p.N1;
  if (threadIdx.x == 0) {
    int p0, Pr;
    prefix_of(p, r, p0, Pr, false);  // the same clamped extent the attention kernels use
    const int nn = p.num_nodes ? p.num_nodes[r] : p.N;
    int pos = -1;
    if (nn >= 0 && nn <= p.N) {
      if (s == 0) {
        pos = Pr;
      } else if (s - 1 < nn) {
        int cur = s - 1, d = 1;
        for (int it = 0; it <= p.N; ++it) {
          const int par = p.parents ? p.parents[(size_t)r * p.N + cur] : cur - 1;
          if (par < -1 || par >= cur) { d = -1; break; }
          if (par < 0) break;
          ++d;
          cur = par;
        }
        pos = d < 0 ? -1 : Pr + d;
        if (d < 0 && p.status) atomicOr(p.status, (uint32_t)AURORA_STATUS_STRUCTURE);
      }
    } else if (p.status) {
      atomicOr(p.status, (uint32_t)AURORA_STATUS_STRUCTURE);
    }
    s_pos = pos;
  }
  __syncthreads();
  const int pos = s_pos;
  if (pos < 0) return;  // padded / malformed row: left unrotated
  const int half = dh >> 1;
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    const double w = exp2(-(2.0 * i / dh) * log2_theta);
    double sn, cs;
    sincos(static_cast<double>(pos) * w, &sn, &cs);
    s_cos[i] = static_cast<float>(cs);
    s_sin[i] = static_cast<float>(inverse ? -sn : sn);
  }
  __syncthreads();
  auto rot = [&](auto* base, int heads) {
    for (int e = threadIdx.x; e < heads * half; e += blockDim.x) {
      const int h = e / half, i = e - h * half;
      auto* x = base + ((size_t)row * heads + h) * dh;
      const float a = static_cast<float>(x[i]), b = static_cast<float>(x[i + half]);
      const float c = s_cos[i], sn = s_sin[i];
      x[i] = static_cast<std::remove_reference_t<decltype(x[i])>>(a * c - b * sn);
      x[i + half] = static_cast<std::remove_reference_t<decltype(x[i])>>(b * c + a * sn);
    }
  };
  if (Q) rot(Q, p.Hq);
  if (Kt) rot(Kt, p.Hkv);
}

// ------------------------------------------------------------------------------ host
struct TaLaunch {
  int Gc, nchunk, nw;
};

bool misaligned16(std::initializer_list<const void*> ps) {
  for (const void* q : ps)
    if (reinterpret_cast<uintptr_t>(q) & 15) return true;
  return false;
}

aurora_status_t ta_check(const aurora_tree_attn_t* ta) {
  if (!ta || !ta->prefix_off) return AURORA_ERR_INVALID_ARG;
  if (ta->R < 1 || ta->N < 1 || ta->Hq < 1 || ta->Hkv < 1 || ta->max_prefix < 0) return AURORA_ERR_INVALID_ARG;
  if (ta->Hq % ta->Hkv) return AURORA_ERR_INVALID_ARG;
  if (ta->R > 65535 || ta->Hkv > 65535) return AURORA_ERR_UNSUPPORTED;
  if (ta->dh != D || ta->N > AURORA_MAX_NODES) return AURORA_ERR_UNSUPPORTED;
  if ((ta->Hq / ta->Hkv) * (ta->N + 1) > kMaxRowsReq) return AURORA_ERR_UNSUPPORTED;
  return AURORA_OK;
}

TaParams ta_params(const aurora_tree_attn_t* ta, TaLaunch& L) {
  TaParams p{};
  p.R = ta->R;
  p.N = ta->N;
  p.N1 = ta->N + 1;
  p.Hq = ta->Hq;
  p.Hkv = ta->Hkv;
  p.G = ta->Hq / ta->Hkv;
  p.max_prefix = ta->max_prefix;
  p.prefix_total = static_cast<int>(std::min<int64_t>(ta->prefix_total, INT32_MAX));
  p.scale = ta->scale > 0.f ? ta->scale : 1.f / sqrtf((float)D);
  p.c2 = p.scale * kLog2e;
  p.prefix_off = ta->prefix_off;
  p.parents = ta->parents;
  p.num_nodes = ta->num_nodes;
  p.status = ta->status;
  L.Gc = std::min(p.G, kMaxRowsCta / p.N1);
  L.nchunk = (p.G + L.Gc - 1) / L.Gc;
  L.nw = (L.Gc * p.N1 + 15) / 16;
  p.Gc = L.Gc;
  return p;
}

size_t smem_fwd(int nw) { return (size_t)nw * 16 * ROWB + 2 * kFwdST * kFwdNK * ROWB + 40 * 8; }
size_t smem_dq(int nw) { return (size_t)2 * nw * 16 * ROWB + 2 * kDqST * kDqNK * ROWB + 40 * 8; }
constexpr size_t kSmemFused = 2 * 128 * ROWB + 2 * kFbST * kFbNK * ROWB + 2 * 128 * kFbRowB + 40 * 8;
constexpr size_t kSmemDkdv = 2 * KT2 * ROWB + 4 * QC * ROWB + 40 * 8 + kMaxRowsReq * 16 + 4 * (kMaxRowsReq / QC);

}  // namespace
}  // namespace aur

using namespace aur;

extern "C" aurora_status_t aurora_tree_attn_fwd(const aurora_tree_attn_t* ta, const void* Q, const void* Kt,
                                                const void* Vt, const void* Kp, const void* Vp, void* O, float* lse,
                                                void* stream) {
  aurora_status_t st = ta_check(ta);
  if (st != AURORA_OK) return st;
  if (!Q || !Kt || !Vt || !O || !lse) return AURORA_ERR_INVALID_ARG;
  if (ta->max_prefix > 0 && (!Kp || !Vp)) return AURORA_ERR_INVALID_ARG;
  if (misaligned16({Q, Kt, Vt, Kp, Vp, O})) return AURORA_ERR_INVALID_ARG;  // 16-B vector / TMA access
  TaLaunch L;
  TaParams p = ta_params(ta, L);
  p.Q = (const uint16_t*)Q;
  p.Kt = (const uint16_t*)Kt;
  p.Vt = (const uint16_t*)Vt;
  p.Kp = (const uint16_t*)Kp;
  p.Vp = (const uint16_t*)Vp;
  p.Oout = (uint16_t*)O;
  p.lse_out = lse;
  cudaStream_t s = (cudaStream_t)stream;
  const int tcmode = opt_tree_fwd_tc();
  if (tcmode && p.G * p.N1 <= 128) {
    TaTcMaps maps;
    const uint64_t rows_t = (uint64_t)p.R * p.N1;
    const uint64_t ptot = ta->prefix_total > 0 ? (uint64_t)ta->prefix_total : 1;
    const void* kp = ta->prefix_total > 0 ? Kp : Kt;
    const void* vp = ta->prefix_total > 0 ? Vp : Vt;
    bool ok = make_tmap_bf16_3d(&maps.Q, Q, D, p.Hq, rows_t, D, (uint64_t)p.Hq * D, 64, p.G, p.N1) &&
              make_tmap_bf16_3d(&maps.Kp, kp, D, p.Hkv, ptot, D, (uint64_t)p.Hkv * D, 64, 1, kTcNK) &&
              make_tmap_bf16_3d(&maps.Vp, vp, D, p.Hkv, ptot, D, (uint64_t)p.Hkv * D, 64, 1, kTcNK) &&
              make_tmap_bf16_3d(&maps.Kt, Kt, D, p.Hkv, rows_t, D, (uint64_t)p.Hkv * D, 64, 1, kTcNK) &&
              make_tmap_bf16_3d(&maps.Vt, Vt, D, p.Hkv, rows_t, D, (uint64_t)p.Hkv * D, 64, 1, kTcNK);
    if (!ok) return AURORA_ERR_CUDA;
    static bool tattr = false;
    if (!tattr) {
      cudaFuncSetAttribute(k_ta_fwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemTc);
      cudaFuncSetAttribute(k_ta_fwd_tc2<2, 2, 2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)TcPlan<2, 2, 2, 1>::kSmem);
      cudaFuncSetAttribute(k_ta_fwd_tc2<1, 4, 4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)TcPlan<1, 4, 4, 2>::kSmem);
      tattr = true;
    }
    const int work = p.R * p.Hkv;
    prof_begin(PH_TREE_FWD_TC, s);
    if (tcmode == 1)
      k_ta_fwd_tc<<<std::min(work, kNumSMs), kTcThreads, kSmemTc, s>>>(maps, p);
    else if (tcmode == 2)
      k_ta_fwd_tc2<2, 2, 2, 1><<<std::min((work + 1) / 2, kNumSMs), TcPlan<2, 2, 2, 1>::kThreads,
                                  TcPlan<2, 2, 2, 1>::kSmem, s>>>(maps, p);
    else
      k_ta_fwd_tc2<1, 4, 4, 2><<<std::min(work, kNumSMs), TcPlan<1, 4, 4, 2>::kThreads,
                                  TcPlan<1, 4, 4, 2>::kSmem, s>>>(maps, p);
    count_launch();
    prof_end(PH_TREE_FWD_TC, s);
    return cudaGetLastError() == cudaSuccess ? AURORA_OK : AURORA_ERR_CUDA;
  }
  const size_t sm = smem_fwd(L.nw);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_ta_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_fwd(7));
    cudaFuncSetAttribute(k_ta_fwd, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr = true;
  }
  prof_begin(PH_TREE_FWD, s);
  k_ta_fwd<<<dim3(p.R, p.Hkv, L.nchunk), L.nw * 32, sm, s>>>(p);
  count_launch();
  prof_end(PH_TREE_FWD, s);
  return cudaGetLastError() == cudaSuccess ? AURORA_OK : AURORA_ERR_CUDA;
}

extern "C" size_t aurora_tree_attn_workspace_size(const aurora_tree_attn_t* ta) {
  if (!ta) return 0;
  return (size_t)ta->R * (ta->N + 1) * ta->Hq * sizeof(float) + 256;
}

extern "C" aurora_status_t aurora_tree_attn_bwd(const aurora_tree_attn_t* ta, const void* Q, const void* Kt,
                                                const void* Vt, const void* Kp, const void* Vp, const void* O,
                                                const float* lse, const void* dO, float* dQ, void* dKt, void* dVt,
                                                void* dKp, void* dVp, void* ws, size_t ws_bytes, void* stream) {
  aurora_status_t st = ta_check(ta);
  if (st != AURORA_OK) return st;
  if (!Q || !Kt || !Vt || !O || !lse || !dO || !dQ || !dKt || !dVt) return AURORA_ERR_INVALID_ARG;
  if (ta->max_prefix > 0 && (!Kp || !Vp || !dKp || !dVp)) return AURORA_ERR_INVALID_ARG;
  if (misaligned16({Q, Kt, Vt, Kp, Vp, O, dO, dQ, dKt, dVt, dKp, dVp})) return AURORA_ERR_INVALID_ARG;
  if (!ws || ws_bytes < aurora_tree_attn_workspace_size(ta)) return AURORA_ERR_WORKSPACE;
  TaLaunch L;
  TaParams p = ta_params(ta, L);
  p.Q = (const uint16_t*)Q;
  p.Kt = (const uint16_t*)Kt;
  p.Vt = (const uint16_t*)Vt;
  p.Kp = (const uint16_t*)Kp;
  p.Vp = (const uint16_t*)Vp;
  p.O = (const uint16_t*)O;
  p.dO = (const uint16_t*)dO;
  p.lse = lse;
  p.Dsum = (const float*)ws;
  p.dQ = dQ;
  p.dKt = (uint16_t*)dKt;
  p.dVt = (uint16_t*)dVt;
  p.dKp = (uint16_t*)dKp;
  p.dVp = (uint16_t*)dVp;
  cudaStream_t s = (cudaStream_t)stream;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_ta_bwd_dq, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_dq(7));
    cudaFuncSetAttribute(k_ta_bwd_dkdv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemDkdv);
    cudaFuncSetAttribute(k_ta_bwd_dq, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
#ifndef TA_NO_DKDV_CARVEOUT
    cudaFuncSetAttribute(k_ta_bwd_dkdv, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
#endif
    attr = true;
  }
  const int64_t n_rows = (int64_t)p.R * p.N1 * p.Hq;
  if (p.G * p.N1 <= 128 && opt_tree_bwd_tc() && !opt_tree_bwd_split()) {
    TaBwdMaps maps;
    const uint64_t rows_t = (uint64_t)p.R * p.N1;
    const uint64_t ptot = ta->prefix_total > 0 ? (uint64_t)ta->prefix_total : 1;
    const void* kp = ta->prefix_total > 0 ? Kp : Kt;
    const void* vp = ta->prefix_total > 0 ? Vp : Vt;
    bool ok = make_tmap_bf16_3d(&maps.Q, Q, D, p.Hq, rows_t, D, (uint64_t)p.Hq * D, 64, p.G, p.N1) &&
              make_tmap_bf16_3d(&maps.dO, dO, D, p.Hq, rows_t, D, (uint64_t)p.Hq * D, 64, p.G, p.N1) &&
              make_tmap_bf16_3d(&maps.Kp, kp, D, p.Hkv, ptot, D, (uint64_t)p.Hkv * D, 64, 1, kT2NK) &&
              make_tmap_bf16_3d(&maps.Vp, vp, D, p.Hkv, ptot, D, (uint64_t)p.Hkv * D, 64, 1, kT2NK) &&
              make_tmap_bf16_3d(&maps.Kt, Kt, D, p.Hkv, rows_t, D, (uint64_t)p.Hkv * D, 64, 1, kT2NK) &&
              make_tmap_bf16_3d(&maps.Vt, Vt, D, p.Hkv, rows_t, D, (uint64_t)p.Hkv * D, 64, 1, kT2NK);
    if (!ok) return AURORA_ERR_CUDA;
    static bool tattr = false;
    if (!tattr) {
      cudaFuncSetAttribute(k_ta_bwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemTb);
      tattr = true;
    }
    const int work = p.R * p.Hkv;
    prof_begin(PH_TREE_BWD_FUSED, s);
    k_ta_bwd_tc<<<std::min(work, kNumSMs), 64 + kTbCompute, kSmemTb, s>>>(maps, p);  // D formed in-kernel
    prof_end(PH_TREE_BWD_FUSED, s);
    count_launch(1);
    return cudaGetLastError() == cudaSuccess ? AURORA_OK : AURORA_ERR_CUDA;
  }
  if (p.G * p.N1 <= 128 && !opt_tree_bwd_split()) {
    static bool fattr = false;
    if (!fattr) {
      cudaFuncSetAttribute(k_ta_bwd_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemFused);
      fattr = true;
    }
    prof_begin(PH_TREE_BWD_FUSED, s);
    k_ta_dsum<<<(unsigned)((n_rows + 7) / 8), 256, 0, s>>>(p.O, p.dO, (float*)ws, n_rows);
    k_ta_bwd_fused<<<dim3(p.R, p.Hkv), 256, kSmemFused, s>>>(p);
    prof_end(PH_TREE_BWD_FUSED, s);
    count_launch(2);
  } else {
    prof_begin(PH_TREE_BWD_DQ, s);
    k_ta_dsum<<<(unsigned)((n_rows + 7) / 8), 256, 0, s>>>(p.O, p.dO, (float*)ws, n_rows);
    k_ta_bwd_dq<<<dim3(p.R, p.Hkv, L.nchunk), L.nw * 32, smem_dq(L.nw), s>>>(p);
    prof_end(PH_TREE_BWD_DQ, s);
    prof_begin(PH_TREE_BWD_DKDV, s);
    const int ktiles = (ta->max_prefix + p.N1 + KT2 - 1) / KT2;
    k_ta_bwd_dkdv<<<dim3(ktiles, p.Hkv, p.R), 256, kSmemDkdv, s>>>(p);
    prof_end(PH_TREE_BWD_DKDV, s);
    count_launch(3);
  }
  return cudaGetLastError() == cudaSuccess ? AURORA_OK : AURORA_ERR_CUDA;
}

extern "C" aurora_status_t aurora_tree_rope(const aurora_tree_attn_t* ta, void* Q, int q_fp32, void* Kt,
                                            int kt_fp32, float theta, int inverse, void* stream) {
  if (!ta || !ta->prefix_off || ta->R < 1 || ta->N < 1 || ta->Hq < 1 || ta->Hkv < 1) return AURORA_ERR_INVALID_ARG;
  if (ta->N > AURORA_MAX_NODES || ta->dh < 2 || ta->dh > 256 || (ta->dh & 1)) return AURORA_ERR_UNSUPPORTED;
  if (!(theta > 1.f)) return AURORA_ERR_INVALID_ARG;
  if (!Q && !Kt) return AURORA_OK;
  TaLaunch L;
  TaParams p = ta_params(ta, L);
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned grid = (unsigned)(ta->R * (ta->N + 1));
  const double l2t = std::log2(static_cast<double>(theta));
  using bf = __nv_bfloat16;
  if (!q_fp32 && !kt_fp32)
    k_ta_rope<bf, bf><<<grid, 128, 0, s>>>(p, (bf*)Q, (bf*)Kt, ta->dh, l2t, inverse);
  else if (q_fp32 && kt_fp32)
    k_ta_rope<float, float><<<grid, 128, 0, s>>>(p, (float*)Q, (float*)Kt, ta->dh, l2t, inverse);
  else if (q_fp32)
    k_ta_rope<float, bf><<<grid, 128, 0, s>>>(p, (float*)Q, (bf*)Kt, ta->dh, l2t, inverse);
  else
    k_ta_rope<bf, float><<<grid, 128, 0, s>>>(p, (bf*)Q, (float*)Kt, ta->dh, l2t, inverse);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? AURORA_OK : AURORA_ERR_CUDA;
}

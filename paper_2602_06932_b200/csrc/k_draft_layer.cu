// k_draft_layer.cu — NEXT F4: the EAGLE-3 draft layer around the tree attention (reading F4-R7).
//
//   g = h3 Wfc^T;  u = [rms(e) w_e ; rms(g) w_h];  q,k,v = u W{q,k,v}^T;  RoPE(q, k) at tree
//   positions;  o = TreeAttention(q, [Kp; k], [Vp; v]);  y = g + o Wo^T;  z = rms(y) w_post;
//   H = y + (silu(z Wg^T) * (z Wu^T)) Wd^T
//   H_out = rms(H) w_final   (EAGLE-3's final norm before the lm_head; the lm_head path's input)
// Dense projections run on the library's own tcgen05 GEMM engine (k_gemm.cu: TMA-fed
// tcgen05.mma, TMEM accumulators, bf16 / fp32 TMA-store epilogues, residual adds as TMA
// reduce-add); the norms, SwiGLU and their backward passes are the kernels below.  Activations the backward needs are
// kept in the caller's workspace between aurora_draft_layer_fwd and aurora_draft_layer_bwd.
// Deterministic: row-wise reductions in fixed order, norm-weight gradients by a two-stage
// fixed-order column reduction.
#include <cmath>
#include <algorithm>
#include <mutex>

#include "internal.h"

namespace aur {
namespace {

using bf16 = __nv_bfloat16;

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(bf16 x) { return __bfloat162float(x); }

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];  // fixed order
  return t;
}

// 4 consecutive elements (n % 4 == 0, rows 16 B / 8 B aligned)
__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 ld4(const bf16* p) {
  const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
  return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u), __uint_as_float(u.y << 16),
                     __uint_as_float(u.y & 0xFFFF0000u));
}

// y[row, :n] = x * rstd * w (bf16), rstd[row] = (mean(x^2) + eps)^-1/2
template <typename TX>
__global__ void __launch_bounds__(256) k_rms_fwd(const TX* __restrict__ x, int64_t ldx, const float* __restrict__ w,
                                                 float eps, int n, bf16* __restrict__ y, int64_t ldy,
                                                 float* __restrict__ rstd) {
  __shared__ float red[8];
  const int64_t row = blockIdx.x;
  const TX* xr = x + row * ldx;
  float ss = 0.f;
  for (int j = threadIdx.x * 4; j < n; j += blockDim.x * 4) {
    const float4 v = ld4(xr + j);
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  const float r = rsqrtf(block_sum(ss, red) / n + eps);
  for (int j = threadIdx.x * 4; j < n; j += blockDim.x * 4) {
    const float4 v = ld4(xr + j), g = ld4(w + j);
    const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x * r * g.x, v.y * r * g.y);
    const __nv_bfloat162 hi = __floats2bfloat162_rn(v.z * r * g.z, v.w * r * g.w);
    *reinterpret_cast<uint2*>(y + row * ldy + j) =
        make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
  }
  if (threadIdx.x == 0) rstd[row] = r;
}

// dx = add + r (w dy) - x r^3 mean(x w dy)    (add may be null; dx may alias x: each row is
// read completely before it is written)
template <typename TX>
__global__ void __launch_bounds__(256) k_rms_bwd(const TX* x, int64_t ldx, const float* __restrict__ w,
                                                 const float* __restrict__ rstd, const float* __restrict__ dy,
                                                 int64_t ldy, const float* add, int64_t lda,
                                                 float* dx, int64_t lddx, int n) {
  __shared__ float red[8];
  const int64_t row = blockIdx.x;
  const float r = rstd[row];
  float dot = 0.f;
  for (int j = threadIdx.x * 4; j < n; j += blockDim.x * 4) {
    const float4 xv = ld4(x + row * ldx + j), g = ld4(w + j), d4 = ld4(dy + row * ldy + j);
    dot += xv.x * g.x * d4.x + xv.y * g.y * d4.y + xv.z * g.z * d4.z + xv.w * g.w * d4.w;
  }
  const float c = block_sum(dot, red) / n * r * r * r;
  for (int j = threadIdx.x * 4; j < n; j += blockDim.x * 4) {
    const float4 xv = ld4(x + row * ldx + j), g = ld4(w + j), d4 = ld4(dy + row * ldy + j);
    float4 v = make_float4(r * g.x * d4.x - xv.x * c, r * g.y * d4.y - xv.y * c, r * g.z * d4.z - xv.z * c,
                           r * g.w * d4.w - xv.w * c);
    if (add) {
      const float4 a4 = ld4(add + row * lda + j);
      v.x += a4.x; v.y += a4.y; v.z += a4.z; v.w += a4.w;
    }
    *reinterpret_cast<float4*>(dx + row * lddx + j) = v;
  }
}

// dw partials: part[chunk, j] = sum over the chunk's rows of dy * x * rstd (fixed row order)
template <typename TX>
__global__ void __launch_bounds__(256) k_rms_dw_part(const TX* __restrict__ x, int64_t ldx, const float* __restrict__ rstd,
                                                     const float* __restrict__ dy, int64_t ldy, int64_t rows, int n,
                                                     int rows_per_chunk, float* __restrict__ part) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_chunk, r1 = min(rows, r0 + rows_per_chunk);
  float acc = 0.f;
  for (int64_t r = r0; r < r1; ++r) acc += dy[r * ldy + j] * to_f(x[r * ldx + j]) * rstd[r];
  part[(int64_t)blockIdx.y * n + j] = acc;
}
__global__ void k_col_reduce(const float* __restrict__ part, int chunks, int n, float* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  float acc = 0.f;
  for (int c = 0; c < chunks; ++c) acc += part[(int64_t)c * n + j];
  out[j] = acc;
}

__device__ __forceinline__ float silu_f(float a) { return a / (1.f + __expf(-a)); }

// Elementwise passes, 8 elements (16 B of bf16) per thread and iteration; counts are multiples
// of 8 and rows 16 B aligned (d, I multiples of 64).
__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ uint4 pack8(const float* f) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    w[i] = *reinterpret_cast<const uint32_t*>(&h);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__global__ void k_swiglu_fwd(const bf16* __restrict__ a, const bf16* __restrict__ b, bf16* __restrict__ m, int64_t count) {
  const int64_t n8 = count >> 3;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    float fa[8], fb[8], fm[8];
    unpack8(__ldg(reinterpret_cast<const uint4*>(a) + i), fa);
    unpack8(__ldg(reinterpret_cast<const uint4*>(b) + i), fb);
#pragma unroll
    for (int e = 0; e < 8; ++e) fm[e] = silu_f(fa[e]) * fb[e];
    reinterpret_cast<uint4*>(m)[i] = pack8(fm);
  }
}
// da = dm * b * s (1 + a (1 - s)),  db = dm * silu(a)   (bf16: the next GEMMs' operands)
__global__ void k_swiglu_bwd(const bf16* __restrict__ a, const bf16* __restrict__ b, const float* __restrict__ dm,
                             bf16* __restrict__ da, bf16* __restrict__ db, int64_t count) {
  const int64_t n8 = count >> 3;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    float fa[8], fb[8], g[8], oa[8], ob[8];
    unpack8(__ldg(reinterpret_cast<const uint4*>(a) + i), fa);
    unpack8(__ldg(reinterpret_cast<const uint4*>(b) + i), fb);
    const float4 g0 = __ldg(reinterpret_cast<const float4*>(dm) + 2 * i), g1 = __ldg(reinterpret_cast<const float4*>(dm) + 2 * i + 1);
    g[0] = g0.x; g[1] = g0.y; g[2] = g0.z; g[3] = g0.w; g[4] = g1.x; g[5] = g1.y; g[6] = g1.z; g[7] = g1.w;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float s = 1.f / (1.f + __expf(-fa[e]));
      oa[e] = g[e] * fb[e] * s * (1.f + fa[e] * (1.f - s));
      ob[e] = g[e] * fa[e] * s;
    }
    reinterpret_cast<uint4*>(da)[i] = pack8(oa);
    reinterpret_cast<uint4*>(db)[i] = pack8(ob);
  }
}
__global__ void k_f2bf(const float* __restrict__ x, bf16* __restrict__ y, int64_t count) {
  const int64_t n8 = count >> 3;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 u = __ldg(reinterpret_cast<const float4*>(x) + 2 * i), v = __ldg(reinterpret_cast<const float4*>(x) + 2 * i + 1);
    const float f[8] = {u.x, u.y, u.z, u.w, v.x, v.y, v.z, v.w};
    reinterpret_cast<uint4*>(y)[i] = pack8(f);
  }
}

unsigned grid_for(int64_t count) { return (unsigned)std::min<int64_t>((count / 8 + 255) / 256, 148 * 16); }

// ---- dense projections on the library's tcgen05 engine (k_gemm.cu), row-major tensors:
//   C[M, N] (+)= A B^T with A bf16 [M, K] (a_mn: stored as [K, M]) and B bf16 [N, K]
//   (b_mn: stored as [K, N]); C bf16 (TMA bulk-store epilogue) or fp32 (TMA store, or TMA
//   reduce-add when accumulating: the residual adds).  fp32 GEMMs whose tile count leaves
//   SMs idle split K into ordered fp32 partials (split_ws) reduced by k_splitk_reduce.
struct Eng {
  cudaStream_t s;
  float* split_ws;
  int64_t split_elems;
};
bool eng_gemm(const Eng& E, const bf16* A, int64_t lda, bool a_mn, const bf16* B, int64_t ldb, bool b_mn, void* C,
              int64_t ldc, bool out_bf16, bool accumulate, int64_t M, int64_t N, int64_t K) {
  const int pr = (M % 256 == 0 || M >= 4096) ? 2 : 1;
  CUtensorMap ta, tb, tc;
  bool ok = a_mn ? make_tmap_bf16(&ta, A, M, K, lda, 64, 64) : make_tmap_bf16(&ta, A, K, M, lda, 64, BM);
  ok = ok && (b_mn ? make_tmap_bf16(&tb, B, N, K, ldb, 64, 64) : make_tmap_bf16(&tb, B, K, N, ldb, 64, BN / pr));
  if (!ok) return false;
  GemmArgs g{};
  g.m_tiles = static_cast<int32_t>((M + BM * pr - 1) / (BM * pr));
  g.n_tiles = static_cast<int32_t>((N + BN - 1) / BN);
  g.kb_total = static_cast<int32_t>((K + BK - 1) / BK);
  g.M = M;
  g.N = N;
  int splits = 1;
  if (!out_bf16) {  // fill idle SMs with K splits when the output has few tiles
    const int64_t tiles = static_cast<int64_t>(g.m_tiles) * g.n_tiles, slots = kNumSMs / pr;
    if (tiles < slots && ldc == N && (M * N) % 4 == 0) {
      splits = static_cast<int>(std::min<int64_t>({8, slots / tiles, g.kb_total}));
      while (splits > 1 && static_cast<int64_t>(splits) * M * N > E.split_elems) --splits;
    }
  }
  // grouped raster when both operands are large: keep a group of one side's blocks in L2 (~48 MB)
  // while the other side sweeps; pick the side with less HBM re-reading
  {
    const double l2 = 48.0 * (1 << 20), ablk = 2.0 * BM * pr * K, bblk = 2.0 * BN * K;
    const double atot = 2.0 * M * K, btot = 2.0 * N * K;
    if (atot + btot > l2) {
      const int gm = static_cast<int>(std::max(1.0, std::min<double>(g.m_tiles, (l2 - bblk) / ablk)));
      const int gn = static_cast<int>(std::max(1.0, std::min<double>(g.n_tiles, (l2 - ablk) / bblk)));
      const double cm = atot + btot * std::ceil(static_cast<double>(g.m_tiles) / gm);
      const double cn = btot + atot * std::ceil(static_cast<double>(g.n_tiles) / gn);
      g.group = cm <= cn ? gm : gn;
      g.group_on_n = cm <= cn ? 0 : 1;
    }
  }
  g.kb_per_split = (g.kb_total + splits - 1) / splits;
  g.splits = (g.kb_total + g.kb_per_split - 1) / g.kb_per_split;
  splits = g.splits;
  if (out_bf16) {
    if (accumulate || !make_tmap_bf16_out(&tc, C, N, M, ldc)) return false;
    return launch_umma_gemm(EPI_STORE_BF16, a_mn, b_mn, ta, tb, g, E.s, &tc, pr) == cudaSuccess;
  }
  if (splits > 1) {
    g.out = E.split_ws;
    g.ld_out = N;
    g.split_stride = M * N;
    if (!make_tmap_f32_out(&tc, E.split_ws, N, M, N, splits, M * N)) return false;
    if (launch_umma_gemm(EPI_STORE_F32, a_mn, b_mn, ta, tb, g, E.s, &tc, pr) != cudaSuccess) return false;
    return launch_splitk_reduce(E.split_ws, splits, M * N, static_cast<float*>(C), accumulate ? 1 : 0, E.s) ==
           cudaSuccess;
  }
  g.out = static_cast<float*>(C);
  g.ld_out = ldc;
  g.accumulate = accumulate ? 1 : 0;
  const bool tmc = make_tmap_f32_out(&tc, C, N, M, ldc, 1, 0);
  return launch_umma_gemm(EPI_STORE_F32, a_mn, b_mn, ta, tb, g, E.s, tmc ? &tc : nullptr, pr) == cudaSuccess;
}
// Y[M,N] (+)= X[M,K] W[N,K]^T          (nn.Linear forward)
bool gemm_xwt(const Eng& E, const bf16* X, const bf16* W, void* Y, bool y_f32, int M, int N, int K, bool acc) {
  return eng_gemm(E, X, K, false, W, K, false, Y, N, !y_f32, acc, M, N, K);
}
// dX[M,K] (+)= dY[M,N] W[N,K]          (input gradient; W read as the MN-major B operand)
bool gemm_dyw(const Eng& E, const bf16* dY, const bf16* W, void* dX, bool f32, int M, int N, int K, bool acc) {
  return eng_gemm(E, dY, N, false, W, K, true, dX, K, !f32, acc, M, K, N);
}
// dW[N,K] = dY[M,N]^T X[M,K]           (weight gradient, f32; both operands MN-major, K = M)
bool gemm_dw(const Eng& E, const bf16* dY, const bf16* X, float* dW, int M, int N, int K) {
  return eng_gemm(E, dY, N, true, X, K, true, dW, K, false, false, N, K, M);
}

// Workspace layout (bytes), shared by fwd (writes the saved activations) and bwd.
struct DlWs {
  float *g, *rs_e, *rs_h, *lse, *y, *rs_p, *f1, *f2, *part, *dq, *hout, *rs_f, *split;
  int64_t split_elems;
  bf16 *u, *q, *k, *v, *o, *z, *a, *b, *m, *b1, *b2, *b3, *dkt, *dvt;
  uint8_t* ta_ws;
  size_t ta_ws_bytes;
};
template <typename T>
T* take(uint8_t*& p, size_t n) {
  p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
  T* r = reinterpret_cast<T*>(p);
  p += n * sizeof(T);
  return r;
}
size_t carve(const aurora_draft_layer_t* L, uint8_t* base, DlWs* w) {
  const int64_t M = (int64_t)L->ta.R * (L->ta.N + 1), d = L->d, I = L->I;
  const int64_t qd = (int64_t)L->ta.Hq * L->ta.dh, kd = (int64_t)L->ta.Hkv * L->ta.dh;
  const int64_t wide = std::max<int64_t>({3 * d, I, qd, 2 * d});
  uint8_t* p = base;
  DlWs t{};
  t.g = take<float>(p, M * d);
  t.rs_e = take<float>(p, M);
  t.rs_h = take<float>(p, M);
  t.lse = take<float>(p, M * L->ta.Hq);
  t.y = take<float>(p, M * d);
  t.rs_p = take<float>(p, M);
  t.f1 = take<float>(p, M * wide);
  t.f2 = take<float>(p, M * wide);
  t.part = take<float>(p, (int64_t)64 * wide);
  t.dq = take<float>(p, M * qd);
  t.hout = take<float>(p, M * d);
  t.rs_f = take<float>(p, M);
  t.split_elems = std::min<int64_t>(M * wide * 4, int64_t(8) * 4096 * 4096);  // split-K partials
  t.split = take<float>(p, t.split_elems);
  t.u = take<bf16>(p, M * 2 * d);
  t.q = take<bf16>(p, M * qd);
  t.k = take<bf16>(p, M * kd);
  t.v = take<bf16>(p, M * kd);
  t.o = take<bf16>(p, M * qd);
  t.z = take<bf16>(p, M * d);
  t.a = take<bf16>(p, M * I);
  t.b = take<bf16>(p, M * I);
  t.m = take<bf16>(p, M * I);
  t.b1 = take<bf16>(p, M * wide);
  t.b2 = take<bf16>(p, M * wide);
  t.b3 = take<bf16>(p, M * wide);
  t.dkt = take<bf16>(p, M * kd);
  t.dvt = take<bf16>(p, M * kd);
  t.ta_ws_bytes = aurora_tree_attn_workspace_size(&L->ta);
  t.ta_ws = take<uint8_t>(p, t.ta_ws_bytes);
  if (w) *w = t;
  return (size_t)(p - base) + 256;
}

template <typename TX>
void rms_dw(cudaStream_t s, const TX* x, int64_t ldx, const float* rstd, const float* dy, int64_t ldy, int64_t rows,
            int n, float* part, float* out) {
  const int chunks = (int)std::min<int64_t>(64, std::max<int64_t>(1, rows / 64));
  const int rpc = (int)((rows + chunks - 1) / chunks);
  k_rms_dw_part<TX><<<dim3((n + 255) / 256, chunks), 256, 0, s>>>(x, ldx, rstd, dy, ldy, rows, n, rpc, part);
  k_col_reduce<<<(n + 255) / 256, 256, 0, s>>>(part, chunks, n, out);
}

aurora_status_t dl_check(const aurora_draft_layer_t* L, const aurora_draft_weights_t* W) {
  if (!L || !W || L->d < 1 || L->I < 1 || L->d % 8 || L->I % 8 || !(L->eps > 0.f)) return AURORA_ERR_INVALID_ARG;
  if (L->ta.dh != 128) return AURORA_ERR_UNSUPPORTED;
  if (!W->Wfc || !W->Wq || !W->Wk || !W->Wv || !W->Wo || !W->Wg || !W->Wu || !W->Wd || !W->we || !W->wh || !W->wpost ||
      !W->wfinal)
    return AURORA_ERR_INVALID_ARG;
  if (L->d % 64 || L->I % 64) return AURORA_ERR_UNSUPPORTED;  // GEMM engine: K multiple of 64 (tails unsupported)
  return AURORA_OK;
}

}  // namespace
}  // namespace aur

using namespace aur;

extern "C" size_t aurora_draft_layer_workspace_size(const aurora_draft_layer_t* L) {
  if (!L) return 0;
  return carve(L, nullptr, nullptr);
}

extern "C" aurora_status_t aurora_draft_layer_fwd(const aurora_draft_layer_t* L, const aurora_draft_weights_t* W,
                                                  const void* h3, const void* e, const void* Kp, const void* Vp,
                                                  void* H, void* ws, size_t ws_bytes, void* stream) {
  aurora_status_t st = dl_check(L, W);
  if (st != AURORA_OK) return st;
  if (!h3 || !e || !H) return AURORA_ERR_INVALID_ARG;
  if (!ws || ws_bytes < aurora_draft_layer_workspace_size(L)) return AURORA_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  DlWs w;
  carve(L, (uint8_t*)ws, &w);
  const int M = L->ta.R * (L->ta.N + 1), d = L->d, I = L->I;
  const int qd = L->ta.Hq * L->ta.dh, kd = L->ta.Hkv * L->ta.dh;
  const bf16 *Wfc = (const bf16*)W->Wfc, *Wq = (const bf16*)W->Wq, *Wk = (const bf16*)W->Wk, *Wv = (const bf16*)W->Wv;
  const bf16 *Wo = (const bf16*)W->Wo, *Wg = (const bf16*)W->Wg, *Wu = (const bf16*)W->Wu, *Wd = (const bf16*)W->Wd;
  const Eng E{s, w.split, w.split_elems};
  bool ok = gemm_xwt(E, (const bf16*)h3, Wfc, w.g, true, M, d, 3 * d, false);                 // g = h3 Wfc^T
  k_rms_fwd<bf16><<<M, 256, 0, s>>>((const bf16*)e, d, W->we, L->eps, d, w.u, 2 * d, w.rs_e);  // u = [rms(e) we ;
  k_rms_fwd<float><<<M, 256, 0, s>>>(w.g, d, W->wh, L->eps, d, w.u + d, 2 * d, w.rs_h);        //      rms(g) wh]
  ok = ok && gemm_xwt(E, w.u, Wq, w.q, false, M, qd, 2 * d, false) &&
       gemm_xwt(E, w.u, Wk, w.k, false, M, kd, 2 * d, false) && gemm_xwt(E, w.u, Wv, w.v, false, M, kd, 2 * d, false);
  if (!ok) return AURORA_ERR_CUDA;
  st = aurora_tree_rope(&L->ta, w.q, 0, w.k, 0, L->theta, 0, s);
  if (st == AURORA_OK) st = aurora_tree_attn_fwd(&L->ta, w.q, w.k, w.v, Kp, Vp, w.o, w.lse, s);
  if (st != AURORA_OK) return st;
  if (cudaMemcpyAsync(w.y, w.g, (size_t)M * d * 4, cudaMemcpyDeviceToDevice, s) != cudaSuccess) return AURORA_ERR_CUDA;
  ok = gemm_xwt(E, w.o, Wo, w.y, true, M, d, qd, true);                                       // y = g + o Wo^T
  k_rms_fwd<float><<<M, 256, 0, s>>>(w.y, d, W->wpost, L->eps, d, w.z, d, w.rs_p);             // z = rms(y) wpost
  ok = ok && gemm_xwt(E, w.z, Wg, w.a, false, M, I, d, false) && gemm_xwt(E, w.z, Wu, w.b, false, M, I, d, false);
  k_swiglu_fwd<<<grid_for((int64_t)M * I), 256, 0, s>>>(w.a, w.b, w.m, (int64_t)M * I);        // m = silu(a) b
  if (cudaMemcpyAsync(w.hout, w.y, (size_t)M * d * 4, cudaMemcpyDeviceToDevice, s) != cudaSuccess) return AURORA_ERR_CUDA;
  ok = ok && gemm_xwt(E, w.m, Wd, w.hout, true, M, d, I, true);                               // h = y + m Wd^T
  k_rms_fwd<float><<<M, 256, 0, s>>>(w.hout, d, W->wfinal, L->eps, d, (bf16*)H, d, w.rs_f);    // H = rms(h) wfinal
  count_launch(5);
  if (!ok) return AURORA_ERR_CUDA;
  return cudaGetLastError() == cudaSuccess ? AURORA_OK : AURORA_ERR_CUDA;
}

extern "C" aurora_status_t aurora_draft_layer_bwd(const aurora_draft_layer_t* L, const aurora_draft_weights_t* W,
                                                  const void* h3, const void* e, const void* Kp, const void* Vp,
                                                  const float* dH, const aurora_draft_grads_t* G, float* dh3,
                                                  float* de, void* dKp, void* dVp, void* ws, size_t ws_bytes,
                                                  void* stream) {
  aurora_status_t st = dl_check(L, W);
  if (st != AURORA_OK) return st;
  if (!h3 || !e || !dH || !G || !dh3 || !de || !G->Wfc || !G->Wq || !G->Wk || !G->Wv || !G->Wo || !G->Wg || !G->Wu ||
      !G->Wd || !G->we || !G->wh || !G->wpost || !G->wfinal)
    return AURORA_ERR_INVALID_ARG;
  if (!ws || ws_bytes < aurora_draft_layer_workspace_size(L)) return AURORA_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  DlWs w;
  carve(L, (uint8_t*)ws, &w);
  const int M = L->ta.R * (L->ta.N + 1), d = L->d, I = L->I;
  const int qd = L->ta.Hq * L->ta.dh, kd = L->ta.Hkv * L->ta.dh;
  const bf16 *Wfc = (const bf16*)W->Wfc, *Wq = (const bf16*)W->Wq, *Wk = (const bf16*)W->Wk, *Wv = (const bf16*)W->Wv;
  const bf16 *Wo = (const bf16*)W->Wo, *Wg = (const bf16*)W->Wg, *Wu = (const bf16*)W->Wu, *Wd = (const bf16*)W->Wd;
  const int64_t MI = (int64_t)M * I, Md = (int64_t)M * d;
  const Eng E{s, w.split, w.split_elems};
  // H = rms(h) wfinal  (dh overwrites h in place: k_rms_bwd reads a row before writing it)
  float* dh = w.hout;
  rms_dw<float>(s, w.hout, d, w.rs_f, dH, d, M, d, w.part, G->wfinal);
  k_rms_bwd<float><<<M, 256, 0, s>>>(w.hout, d, W->wfinal, w.rs_f, dH, d, nullptr, 0, dh, d, d);
  // h = y + m Wd^T
  k_f2bf<<<grid_for(Md), 256, 0, s>>>(dh, w.b1, Md);                                            // b1 = bf16(dh)
  bool ok = gemm_dw(E, w.b1, w.m, G->Wd, M, d, I) && gemm_dyw(E, w.b1, Wd, w.f1, true, M, d, I, false);  // f1 = dm
  k_swiglu_bwd<<<grid_for(MI), 256, 0, s>>>(w.a, w.b, w.f1, w.b2, w.b3, MI);                    // b2 = da, b3 = db
  ok = ok && gemm_dw(E, w.b2, w.z, G->Wg, M, I, d) && gemm_dw(E, w.b3, w.z, G->Wu, M, I, d) &&
       gemm_dyw(E, w.b2, Wg, w.f2, true, M, I, d, false) && gemm_dyw(E, w.b3, Wu, w.f2, true, M, I, d, true);  // f2 = dz
  // z = rms(y) wpost ; dy = dh + rms_bwd
  rms_dw<float>(s, w.y, d, w.rs_p, w.f2, d, M, d, w.part, G->wpost);
  k_rms_bwd<float><<<M, 256, 0, s>>>(w.y, d, W->wpost, w.rs_p, w.f2, d, dh, d, w.f1, d, d);     // f1 = dy
  // y = g + o Wo^T
  k_f2bf<<<grid_for(Md), 256, 0, s>>>(w.f1, w.b1, Md);                                          // b1 = bf16(dy)
  ok = ok && gemm_dw(E, w.b1, w.o, G->Wo, M, d, qd) && gemm_dyw(E, w.b1, Wo, w.b2, false, M, d, qd, false);  // b2 = do
  if (!ok) return AURORA_ERR_CUDA;
  st = aurora_tree_attn_bwd(&L->ta, w.q, w.k, w.v, Kp, Vp, w.o, w.lse, w.b2, w.dq, w.dkt, w.dvt, dKp, dVp, w.ta_ws,
                            w.ta_ws_bytes, s);
  if (st == AURORA_OK) st = aurora_tree_rope(&L->ta, w.dq, 1, w.dkt, 0, L->theta, 1, s);
  if (st != AURORA_OK) return st;
  k_f2bf<<<grid_for((int64_t)M * qd), 256, 0, s>>>(w.dq, w.b3, (int64_t)M * qd);                // b3 = bf16(dq)
  ok = gemm_dw(E, w.b3, w.u, G->Wq, M, qd, 2 * d) && gemm_dw(E, w.dkt, w.u, G->Wk, M, kd, 2 * d) &&
       gemm_dw(E, w.dvt, w.u, G->Wv, M, kd, 2 * d) && gemm_dyw(E, w.b3, Wq, w.f2, true, M, qd, 2 * d, false) &&
       gemm_dyw(E, w.dkt, Wk, w.f2, true, M, kd, 2 * d, true) && gemm_dyw(E, w.dvt, Wv, w.f2, true, M, kd, 2 * d, true);
  // u = [rms(e) we ; rms(g) wh]   (f2 = du [M, 2d])
  rms_dw<bf16>(s, (const bf16*)e, d, w.rs_e, w.f2, 2 * d, M, d, w.part, G->we);
  k_rms_bwd<bf16><<<M, 256, 0, s>>>((const bf16*)e, d, W->we, w.rs_e, w.f2, 2 * d, nullptr, 0, de, d, d);
  rms_dw<float>(s, w.g, d, w.rs_h, w.f2 + d, 2 * d, M, d, w.part, G->wh);
  k_rms_bwd<float><<<M, 256, 0, s>>>(w.g, d, W->wh, w.rs_h, w.f2 + d, 2 * d, w.f1, d, w.f1, d, d);  // f1 = dg
  // g = h3 Wfc^T
  k_f2bf<<<grid_for(Md), 256, 0, s>>>(w.f1, w.b1, Md);
  ok = ok && gemm_dw(E, w.b1, (const bf16*)h3, G->Wfc, M, d, 3 * d) &&
       gemm_dyw(E, w.b1, Wfc, dh3, true, M, d, 3 * d, false);
  count_launch(18);
  if (!ok) return AURORA_ERR_CUDA;
  return cudaGetLastError() == cudaSuccess ? AURORA_OK : AURORA_ERR_CUDA;
}

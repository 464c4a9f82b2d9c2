// k_draft_layer.cu — NEXT F4: the EAGLE-3 draft layer around the tree attention (reading F4-R7).
//
//   g = h3 Wfc^T;  u = [rms(e) w_e ; rms(g) w_h];  q,k,v = u W{q,k,v}^T;  RoPE(q, k) at tree
//   positions;  o = TreeAttention(q, [Kp; k], [Vp; v]);  y = g + o Wo^T;  z = rms(y) w_post;
//   H = y + (silu(z Wg^T) * (z Wu^T)) Wd^T
// Dense projections are plain library GEMMs (cuBLAS, bf16 operands, fp32 accumulation: the
// method-specific arithmetic is the tree attention + RoPE, in k_tree_attn.cu); the norms,
// SwiGLU and their backward passes are the kernels below.  Activations the backward needs are
// kept in the caller's workspace between aurora_draft_layer_fwd and aurora_draft_layer_bwd.
// Deterministic: row-wise reductions in fixed order, norm-weight gradients by a two-stage
// fixed-order column reduction.
#include <cublas_v2.h>

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

// y[row, :n] = x * rstd * w (bf16), rstd[row] = (mean(x^2) + eps)^-1/2
template <typename TX>
__global__ void __launch_bounds__(256) k_rms_fwd(const TX* __restrict__ x, int64_t ldx, const float* __restrict__ w,
                                                 float eps, int n, bf16* __restrict__ y, int64_t ldy,
                                                 float* __restrict__ rstd) {
  __shared__ float red[8];
  const int64_t row = blockIdx.x;
  const TX* xr = x + row * ldx;
  float ss = 0.f;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const float v = to_f(xr[j]);
    ss += v * v;
  }
  const float r = rsqrtf(block_sum(ss, red) / n + eps);
  for (int j = threadIdx.x; j < n; j += blockDim.x) y[row * ldy + j] = __float2bfloat16(to_f(xr[j]) * r * w[j]);
  if (threadIdx.x == 0) rstd[row] = r;
}

// dx = add + r (w dy) - x r^3 mean(x w dy)    (add may be null)
template <typename TX>
__global__ void __launch_bounds__(256) k_rms_bwd(const TX* __restrict__ x, int64_t ldx, const float* __restrict__ w,
                                                 const float* __restrict__ rstd, const float* __restrict__ dy,
                                                 int64_t ldy, const float* __restrict__ add, int64_t lda,
                                                 float* __restrict__ dx, int64_t lddx, int n) {
  __shared__ float red[8];
  const int64_t row = blockIdx.x;
  const float r = rstd[row];
  float dot = 0.f;
  for (int j = threadIdx.x; j < n; j += blockDim.x) dot += to_f(x[row * ldx + j]) * w[j] * dy[row * ldy + j];
  const float c = block_sum(dot, red) / n * r * r * r;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    float v = r * w[j] * dy[row * ldy + j] - to_f(x[row * ldx + j]) * c;
    if (add) v += add[row * lda + j];
    dx[row * lddx + j] = v;
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

__global__ void k_swiglu_fwd(const bf16* __restrict__ a, const bf16* __restrict__ b, bf16* __restrict__ m, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    m[i] = __float2bfloat16(silu_f(__bfloat162float(a[i])) * __bfloat162float(b[i]));
}
// da = dm * b * s (1 + a (1 - s)),  db = dm * silu(a)   (bf16: the next GEMMs' operands)
__global__ void k_swiglu_bwd(const bf16* __restrict__ a, const bf16* __restrict__ b, const float* __restrict__ dm,
                             bf16* __restrict__ da, bf16* __restrict__ db, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const float av = __bfloat162float(a[i]), bv = __bfloat162float(b[i]);
    const float s = 1.f / (1.f + __expf(-av));
    da[i] = __float2bfloat16(dm[i] * bv * s * (1.f + av * (1.f - s)));
    db[i] = __float2bfloat16(dm[i] * av * s);
  }
}
__global__ void k_f2bf(const float* __restrict__ x, bf16* __restrict__ y, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __float2bfloat16(x[i]);
}

unsigned grid_for(int64_t count) { return (unsigned)std::min<int64_t>((count + 255) / 256, 148 * 16); }

// ---- cuBLAS (column-major) wrappers for row-major tensors
cublasHandle_t handle() {
  static cublasHandle_t h = nullptr;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (!h && cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) h = nullptr;
  return h;
}
// Y[M,N] (+)= X[M,K] W[N,K]^T        (Y f32 or bf16)
bool gemm_xwt(cudaStream_t s, const bf16* X, const bf16* W, void* Y, bool y_f32, int M, int N, int K, float beta) {
  cublasHandle_t h = handle();
  if (!h || cublasSetStream(h, s) != CUBLAS_STATUS_SUCCESS) return false;
  const float alpha = 1.f;
  return cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, N, M, K, &alpha, W, CUDA_R_16BF, K, X, CUDA_R_16BF, K, &beta, Y,
                      y_f32 ? CUDA_R_32F : CUDA_R_16BF, N, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT) ==
         CUBLAS_STATUS_SUCCESS;
}
// dX[M,K] (+)= dY[M,N] W[N,K]        (dX f32 or bf16)
bool gemm_dyw(cudaStream_t s, const bf16* dY, const bf16* W, void* dX, bool f32, int M, int N, int K, float beta) {
  cublasHandle_t h = handle();
  if (!h || cublasSetStream(h, s) != CUBLAS_STATUS_SUCCESS) return false;
  const float alpha = 1.f;
  return cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, K, M, N, &alpha, W, CUDA_R_16BF, K, dY, CUDA_R_16BF, N, &beta, dX,
                      f32 ? CUDA_R_32F : CUDA_R_16BF, K, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT) ==
         CUBLAS_STATUS_SUCCESS;
}
// dW[N,K] = dY[M,N]^T X[M,K]          (f32)
bool gemm_dw(cudaStream_t s, const bf16* dY, const bf16* X, float* dW, int M, int N, int K) {
  cublasHandle_t h = handle();
  if (!h || cublasSetStream(h, s) != CUBLAS_STATUS_SUCCESS) return false;
  const float alpha = 1.f, beta = 0.f;
  return cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_T, K, N, M, &alpha, X, CUDA_R_16BF, K, dY, CUDA_R_16BF, N, &beta, dW,
                      CUDA_R_32F, K, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT) == CUBLAS_STATUS_SUCCESS;
}

// Workspace layout (bytes), shared by fwd (writes the saved activations) and bwd.
struct DlWs {
  float *g, *rs_e, *rs_h, *lse, *y, *rs_p, *f1, *f2, *part, *dq;
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
  if (!W->Wfc || !W->Wq || !W->Wk || !W->Wv || !W->Wo || !W->Wg || !W->Wu || !W->Wd || !W->we || !W->wh || !W->wpost)
    return AURORA_ERR_INVALID_ARG;
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
  bool ok = gemm_xwt(s, (const bf16*)h3, Wfc, w.g, true, M, d, 3 * d, 0.f);                    // g = h3 Wfc^T
  k_rms_fwd<bf16><<<M, 256, 0, s>>>((const bf16*)e, d, W->we, L->eps, d, w.u, 2 * d, w.rs_e);  // u = [rms(e) we ;
  k_rms_fwd<float><<<M, 256, 0, s>>>(w.g, d, W->wh, L->eps, d, w.u + d, 2 * d, w.rs_h);        //      rms(g) wh]
  ok = ok && gemm_xwt(s, w.u, Wq, w.q, false, M, qd, 2 * d, 0.f) && gemm_xwt(s, w.u, Wk, w.k, false, M, kd, 2 * d, 0.f) &&
       gemm_xwt(s, w.u, Wv, w.v, false, M, kd, 2 * d, 0.f);
  if (!ok) return AURORA_ERR_CUDA;
  st = aurora_tree_rope(&L->ta, w.q, 0, w.k, 0, L->theta, 0, s);
  if (st == AURORA_OK) st = aurora_tree_attn_fwd(&L->ta, w.q, w.k, w.v, Kp, Vp, w.o, w.lse, s);
  if (st != AURORA_OK) return st;
  if (cudaMemcpyAsync(w.y, w.g, (size_t)M * d * 4, cudaMemcpyDeviceToDevice, s) != cudaSuccess) return AURORA_ERR_CUDA;
  ok = gemm_xwt(s, w.o, Wo, w.y, true, M, d, qd, 1.f);                                        // y = g + o Wo^T
  k_rms_fwd<float><<<M, 256, 0, s>>>(w.y, d, W->wpost, L->eps, d, w.z, d, w.rs_p);             // z = rms(y) wpost
  ok = ok && gemm_xwt(s, w.z, Wg, w.a, false, M, I, d, 0.f) && gemm_xwt(s, w.z, Wu, w.b, false, M, I, d, 0.f);
  k_swiglu_fwd<<<grid_for((int64_t)M * I), 256, 0, s>>>(w.a, w.b, w.m, (int64_t)M * I);        // m = silu(a) b
  if (cudaMemcpyAsync(w.f1, w.y, (size_t)M * d * 4, cudaMemcpyDeviceToDevice, s) != cudaSuccess) return AURORA_ERR_CUDA;
  ok = ok && gemm_xwt(s, w.m, Wd, w.f1, true, M, d, I, 1.f);                                  // H = y + m Wd^T
  k_f2bf<<<grid_for((int64_t)M * d), 256, 0, s>>>(w.f1, (bf16*)H, (int64_t)M * d);
  count_launch(8);
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
      !G->Wd || !G->we || !G->wh || !G->wpost)
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
  // H = y + m Wd^T
  k_f2bf<<<grid_for(Md), 256, 0, s>>>(dH, w.b1, Md);                                           // b1 = bf16(dH)
  bool ok = gemm_dw(s, w.b1, w.m, G->Wd, M, d, I) && gemm_dyw(s, w.b1, Wd, w.f1, true, M, d, I, 0.f);  // f1 = dm
  k_swiglu_bwd<<<grid_for(MI), 256, 0, s>>>(w.a, w.b, w.f1, w.b2, w.b3, MI);                    // b2 = da, b3 = db
  ok = ok && gemm_dw(s, w.b2, w.z, G->Wg, M, I, d) && gemm_dw(s, w.b3, w.z, G->Wu, M, I, d) &&
       gemm_dyw(s, w.b2, Wg, w.f2, true, M, I, d, 0.f) && gemm_dyw(s, w.b3, Wu, w.f2, true, M, I, d, 1.f);  // f2 = dz
  // z = rms(y) wpost ; dy = dH + rms_bwd
  rms_dw<float>(s, w.y, d, w.rs_p, w.f2, d, M, d, w.part, G->wpost);
  k_rms_bwd<float><<<M, 256, 0, s>>>(w.y, d, W->wpost, w.rs_p, w.f2, d, dH, d, w.f1, d, d);     // f1 = dy
  // y = g + o Wo^T
  k_f2bf<<<grid_for(Md), 256, 0, s>>>(w.f1, w.b1, Md);                                          // b1 = bf16(dy)
  ok = ok && gemm_dw(s, w.b1, w.o, G->Wo, M, d, qd) && gemm_dyw(s, w.b1, Wo, w.b2, false, M, d, qd, 0.f);  // b2 = do
  if (!ok) return AURORA_ERR_CUDA;
  st = aurora_tree_attn_bwd(&L->ta, w.q, w.k, w.v, Kp, Vp, w.o, w.lse, w.b2, w.dq, w.dkt, w.dvt, dKp, dVp, w.ta_ws,
                            w.ta_ws_bytes, s);
  if (st == AURORA_OK) st = aurora_tree_rope(&L->ta, w.dq, 1, w.dkt, 0, L->theta, 1, s);
  if (st != AURORA_OK) return st;
  k_f2bf<<<grid_for((int64_t)M * qd), 256, 0, s>>>(w.dq, w.b3, (int64_t)M * qd);                // b3 = bf16(dq)
  ok = gemm_dw(s, w.b3, w.u, G->Wq, M, qd, 2 * d) && gemm_dw(s, w.dkt, w.u, G->Wk, M, kd, 2 * d) &&
       gemm_dw(s, w.dvt, w.u, G->Wv, M, kd, 2 * d) && gemm_dyw(s, w.b3, Wq, w.f2, true, M, qd, 2 * d, 0.f) &&
       gemm_dyw(s, w.dkt, Wk, w.f2, true, M, kd, 2 * d, 1.f) && gemm_dyw(s, w.dvt, Wv, w.f2, true, M, kd, 2 * d, 1.f);
  // u = [rms(e) we ; rms(g) wh]   (f2 = du [M, 2d])
  rms_dw<bf16>(s, (const bf16*)e, d, w.rs_e, w.f2, 2 * d, M, d, w.part, G->we);
  k_rms_bwd<bf16><<<M, 256, 0, s>>>((const bf16*)e, d, W->we, w.rs_e, w.f2, 2 * d, nullptr, 0, de, d, d);
  rms_dw<float>(s, w.g, d, w.rs_h, w.f2 + d, 2 * d, M, d, w.part, G->wh);
  k_rms_bwd<float><<<M, 256, 0, s>>>(w.g, d, W->wh, w.rs_h, w.f2 + d, 2 * d, w.f1, d, w.f1, d, d);  // f1 = dg
  // g = h3 Wfc^T
  k_f2bf<<<grid_for(Md), 256, 0, s>>>(w.f1, w.b1, Md);
  ok = ok && gemm_dw(s, w.b1, (const bf16*)h3, G->Wfc, M, d, 3 * d) &&
       gemm_dyw(s, w.b1, Wfc, dh3, true, M, d, 3 * d, 0.f);
  count_launch(16);
  if (!ok) return AURORA_ERR_CUDA;
  return cudaGetLastError() == cudaSuccess ? AURORA_OK : AURORA_ERR_CUDA;
}

// k_optim.cu — NEXT F3: the AdamW step on the fp32 master lm_head (P:487-489, P:495,
// Table 3).  HBM-bound streaming: 4 B/element for the norm pass, 30 B/element
// for the update (read dW, m, v, W; write m, v, W fp32 and the bf16 copy).
//
//   k_sumsq_partial  grid-stride float4 sum of squares, one partial per CTA (fixed
//                    assignment of elements to CTAs and a fixed shuffle/warp order)
//   k_sumsq_final    one CTA: ordered sum of the partials (+ extra_sq) -> norm^2
//   k_adamw          grid-stride float4 update; the clip coefficient min(1, max/(|g|+1e-6))
//                    and the bias corrections are computed per thread from device scalars
#include <cmath>

#include "internal.h"

namespace aur {

constexpr int kOptBlocks = 4 * kNumSMs;  // persistent grid for the streaming passes
constexpr int kOptThreads = 256;

__global__ void __launch_bounds__(kOptThreads) k_sumsq_partial(const float4* __restrict__ g, int64_t n4,
                                                               float* __restrict__ partial) {
  float acc = 0.f;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kOptThreads + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * kOptThreads) {
    const float4 x = __ldg(g + i);
    acc = fmaf(x.x, x.x, acc);
    acc = fmaf(x.y, x.y, acc);
    acc = fmaf(x.z, x.z, acc);
    acc = fmaf(x.w, x.w, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ float red[kOptThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < kOptThreads / 32; ++w) t += red[w];
    partial[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kOptThreads) k_sumsq_final(const float* __restrict__ partial, int nparts,
                                                             const float* __restrict__ extra_sq, float* __restrict__ out) {
  __shared__ float red[kOptThreads];
  float t = 0.f;
  for (int i = threadIdx.x; i < nparts; i += kOptThreads) t += partial[i];
  red[threadIdx.x] = t;
  __syncthreads();
  for (int st = kOptThreads / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0] + (extra_sq ? extra_sq[0] : 0.f);
}

__global__ void __launch_bounds__(kOptThreads) k_adamw(float4* __restrict__ W, uint2* __restrict__ Wb,
                                                       float4* __restrict__ m, float4* __restrict__ v,
                                                       const float4* __restrict__ g, int64_t n4,
                                                       const float* __restrict__ norm_sq, float* __restrict__ grad_norm,
                                                       AdamwScalars c) {
  const float norm = sqrtf(norm_sq[0]);
  const float clip = (c.max_norm > 0.f) ? fminf(1.f, c.max_norm / (norm + 1e-6f)) : 1.f;
  if (grad_norm && blockIdx.x == 0 && threadIdx.x == 0) grad_norm[0] = norm;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kOptThreads + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * kOptThreads) {
    float4 gi = __ldg(g + i);
    float4 mi = m[i], vi = v[i], wi = W[i];
    float* gp = &gi.x;
    float* mp = &mi.x;
    float* vp = &vi.x;
    float* wp = &wi.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float gg = gp[e] * clip;
      mp[e] = fmaf(c.beta1, mp[e], (1.f - c.beta1) * gg);
      vp[e] = fmaf(c.beta2, vp[e], (1.f - c.beta2) * gg * gg);
      const float denom = sqrtf(vp[e]) * c.inv_sqrt_bc2 + c.eps;
      wp[e] = wp[e] * c.decay - c.step_size * (mp[e] / denom);
    }
    m[i] = mi;
    v[i] = vi;
    W[i] = wi;
    if (Wb) {
      const __nv_bfloat162 lo = __floats2bfloat162_rn(wi.x, wi.y);
      const __nv_bfloat162 hi = __floats2bfloat162_rn(wi.z, wi.w);
      Wb[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
    }
  }
}

int adamw_partials() { return kOptBlocks; }

cudaError_t launch_sum_partials(const float* partials, int nparts, const float* extra_sq, float* out, cudaStream_t s) {
  k_sumsq_final<<<1, kOptThreads, 0, s>>>(partials, nparts, extra_sq, out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_sumsq(const float* g, int64_t n, const float* extra_sq, float* partials, float* norm_sq,
                         cudaStream_t s) {
  k_sumsq_partial<<<kOptBlocks, kOptThreads, 0, s>>>(reinterpret_cast<const float4*>(g), n / 4, partials);
  count_launch();
  k_sumsq_final<<<1, kOptThreads, 0, s>>>(partials, kOptBlocks, extra_sq, norm_sq);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_adamw(float* W, void* Wb, float* m, float* v, const float* g, int64_t n, const float* norm_sq,
                         float* grad_norm, const AdamwScalars& c, cudaStream_t s) {
  k_adamw<<<kOptBlocks, kOptThreads, 0, s>>>(reinterpret_cast<float4*>(W), reinterpret_cast<uint2*>(Wb),
                                             reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v),
                                             reinterpret_cast<const float4*>(g), n / 4, norm_sq, grad_norm, c);
  count_launch();
  return cudaGetLastError();
}

}  // namespace aur

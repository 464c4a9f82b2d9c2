// k_optim.cu — NEXT F3: the AdamW step on the fp32 master lm_head (P:487-489, P:495,
// Table 3).  HBM-bound streaming: 4 B/element for the norm pass, 30 B/element
// for the update (read dW, m, v, W; write m, v, W fp32 and the bf16 copy).
//
//   k_sumsq_partial  grid-stride float4 sum of squares, one partial per CTA (fixed
//                    assignment of elements to CTAs and a fixed shuffle/warp order)
//   k_sumsq_final    one CTA: ordered sum of the partials -> norm^2 of this rank's shard
//                    (the VP / DP allreduce of that scalar follows on the host side)
//   k_adamw_prep     one thread: the step (host value, or the device counter in the
//                    optimizer workspace, incremented here so a replayed CUDA graph
//                    advances it), warm-up LR, bias corrections, and the clip coefficient
//                    min(1, max/(|g|+1e-6)) with |g|^2 = allreduced norm^2 + extra_sq (the
//                    other parameter groups, added once, after the allreduce)
//   k_adamw          grid-stride float4 update reading those device scalars
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
                                                             float* __restrict__ out) {
  __shared__ float red[kOptThreads];
  float t = 0.f;
  for (int i = threadIdx.x; i < nparts; i += kOptThreads) t += partial[i];
  red[threadIdx.x] = t;
  __syncthreads();
  for (int st = kOptThreads / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

// torch.optim.AdamW: W <- W (1 - lr_t wd) - lr_t/(1-b1^t) m / (sqrt(v)/sqrt(1-b2^t) + eps)
__global__ void k_adamw_prep(const float* __restrict__ norm_sq, const float* __restrict__ extra_sq, AdamwHyper h,
                             int64_t host_step, int64_t* __restrict__ step_dev, float* __restrict__ sc,
                             float* __restrict__ grad_norm) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t t = host_step;
  if (t <= 0) {
    t = step_dev[0] + 1;
    step_dev[0] = t;
  }
  const double lr_t = (h.warmup > 0 && t < h.warmup) ? static_cast<double>(h.lr) * static_cast<double>(t) / h.warmup
                                                      : static_cast<double>(h.lr);
  const double bc1 = 1.0 - pow(static_cast<double>(h.beta1), static_cast<double>(t));
  const double bc2 = 1.0 - pow(static_cast<double>(h.beta2), static_cast<double>(t));
  const float nsq = norm_sq[0] + (extra_sq ? extra_sq[0] : 0.f);
  const float norm = sqrtf(nsq);
  sc[0] = (h.max_norm > 0.f) ? fminf(1.f, h.max_norm / (norm + 1e-6f)) : 1.f;
  sc[1] = static_cast<float>(lr_t / bc1);
  sc[2] = static_cast<float>(1.0 / sqrt(bc2));
  sc[3] = static_cast<float>(1.0 - lr_t * h.weight_decay);
  sc[4] = h.beta1;
  sc[5] = h.beta2;
  sc[6] = h.eps;
  if (grad_norm) grad_norm[0] = norm;
}

__global__ void __launch_bounds__(kOptThreads) k_adamw(float4* __restrict__ W, uint2* __restrict__ Wb,
                                                       float4* __restrict__ m, float4* __restrict__ v,
                                                       const float4* __restrict__ g, int64_t n4,
                                                       const float* __restrict__ sc) {
  const float clip = sc[0], step_size = sc[1], isb2 = sc[2], decay = sc[3], b1 = sc[4], b2 = sc[5], eps = sc[6];
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
      mp[e] = fmaf(b1, mp[e], (1.f - b1) * gg);
      vp[e] = fmaf(b2, vp[e], (1.f - b2) * gg * gg);
      const float denom = sqrtf(vp[e]) * isb2 + eps;
      wp[e] = wp[e] * decay - step_size * (mp[e] / denom);
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

// <a, b> over n floats (n % 4 == 0): per-CTA partials in fixed order (the Gram-form norm of
// the fused optimizer: ||dZ^T H||_F^2 = sum (dZ dZ^T) .* (H H^T))
__global__ void __launch_bounds__(kOptThreads) k_dot_partial(const float4* __restrict__ a, const float4* __restrict__ b,
                                                             int64_t n4, float* __restrict__ partial) {
  float acc = 0.f;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kOptThreads + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * kOptThreads) {
    const float4 x = __ldg(a + i), y = __ldg(b + i);
    acc = fmaf(x.x, y.x, acc);
    acc = fmaf(x.y, y.y, acc);
    acc = fmaf(x.z, y.z, acc);
    acc = fmaf(x.w, y.w, acc);
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

cudaError_t launch_dot(const float* a, const float* b, int64_t n, float* partials, float* out, cudaStream_t s) {
  k_dot_partial<<<kOptBlocks, kOptThreads, 0, s>>>(reinterpret_cast<const float4*>(a),
                                                   reinterpret_cast<const float4*>(b), n / 4, partials);
  count_launch();
  k_sumsq_final<<<1, kOptThreads, 0, s>>>(partials, kOptBlocks, out);
  count_launch();
  return cudaGetLastError();
}

int adamw_partials() { return kOptBlocks; }

cudaError_t launch_sum_partials(const float* partials, int nparts, float* out, cudaStream_t s) {
  k_sumsq_final<<<1, kOptThreads, 0, s>>>(partials, nparts, out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_sumsq(const float* g, int64_t n, float* partials, float* norm_sq, cudaStream_t s) {
  k_sumsq_partial<<<kOptBlocks, kOptThreads, 0, s>>>(reinterpret_cast<const float4*>(g), n / 4, partials);
  count_launch();
  k_sumsq_final<<<1, kOptThreads, 0, s>>>(partials, kOptBlocks, norm_sq);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_adamw_prep(const float* norm_sq, const float* extra_sq, const AdamwHyper& h, int64_t host_step,
                              int64_t* step_dev, float* sc, float* grad_norm, cudaStream_t s) {
  k_adamw_prep<<<1, 32, 0, s>>>(norm_sq, extra_sq, h, host_step, step_dev, sc, grad_norm);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_adamw(float* W, void* Wb, float* m, float* v, const float* g, int64_t n, const float* sc,
                         cudaStream_t s) {
  k_adamw<<<kOptBlocks, kOptThreads, 0, s>>>(reinterpret_cast<float4*>(W), reinterpret_cast<uint2*>(Wb),
                                             reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v),
                                             reinterpret_cast<const float4*>(g), n / 4, sc);
  count_launch();
  return cudaGetLastError();
}

}  // namespace aur

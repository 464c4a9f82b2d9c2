// k_rows.cu — per-row statistic reductions and small helpers.
//
//   k_reduce_partials  CTA per row: merge the (m, s, u, r) partials of all vocab tiles of
//                      a row (coalesced: partials are [M, n_tiles] row-major) with the
//                      online rule s = s e^{m-m'} + s_t e^{m_t-m'}; fixed strides, shuffle
//                      tree and warp order => deterministic.
//   k_row_combine      thread per row: merge the per-rank (m, s, u, r) in rank order (VP),
//                      lse = m + log s, l = lse - u + H~ = KL(p~ || q) (Eq. 3), w l,
//                      block-ordered partial sums.  F2 reverse-KL rows (NEXT F2):
//                      KL(q || p) = E_q[z - t] - lse + lse_t with E_q[z - t] = r / s,
//                      plus beta (lse - z_y) (NTP) where u = beta z_y.
//   k_loss_sum         one block: ordered sum of the block partials -> loss.
//   k_splitk_reduce    dH = (acc ? dH : 0) + sum_s partial[s], ordered (deterministic).
//   k_dz_rescale       A7 without the recompute GEMM: the forward staged e = exp(z - m_h)
//                      (bf16) in dZ^T; once lse is known, dz = g w exp(m_h - lse) e in
//                      place.  CTA per (vocab tile half h, 1024-row block): the factors
//                      F_m = g w_m exp(m_h,m - lse_m) in shared memory, then 16 B vectors
//                      of 8 rows along dZ^T's contiguous row axis (HBM-bound: 4 B per element).
//   k_dz_support_fix   the support entries: dz_mj = g w_m (exp(z_mj - lse_m) - p~_mj) from
//                      the fp32 logit the forward kept (no cancellation through bf16 e).
#include <cfloat>
#include <climits>

#include "internal.h"
#include "ptx.cuh"

namespace aur {

namespace {
__device__ __forceinline__ void ms_merge(float& m, float& s, float m2, float s2) {
  const float mn = fmaxf(m, m2);
  if (mn == -INFINITY) return;
  s = s * __expf(m - mn) + s2 * __expf(m2 - mn);
  m = mn;
}
// (m, s, r): r = sum e^{z - m} x rescales like s
__device__ __forceinline__ void msr_merge(float& m, float& s, float& r, float m2, float s2, float r2) {
  const float mn = fmaxf(m, m2);
  if (mn == -INFINITY) return;
  const float a = __expf(m - mn), b = __expf(m2 - mn);
  s = s * a + s2 * b;
  r = r * a + r2 * b;
  m = mn;
}
}  // namespace

constexpr int kRedThreads = 128;
// CTA per row: each thread merges a fixed strided subset of the row's partials with four
// independent loads in flight (the chain is latency-bound, not bandwidth-bound), then a
// fixed shuffle tree and the warps in order => deterministic.
__global__ void __launch_bounds__(kRedThreads) k_reduce_partials(const float* __restrict__ pm,
                                                                 const float* __restrict__ ps,
                                                                 const float* __restrict__ pu,
                                                                 const float* __restrict__ pr, int64_t M, int n_tiles,
                                                                 float* __restrict__ msu) {
  const int64_t row = blockIdx.x;
  float m = -INFINITY, s = 0.f, u = 0.f, r = 0.f;
  const int64_t o = row * n_tiles;
  int t = threadIdx.x;
  for (; t + 3 * kRedThreads < n_tiles; t += 4 * kRedThreads) {
    float mm[4], ss[4], uu[4], rr[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      mm[i] = __ldg(pm + o + t + i * kRedThreads);
      ss[i] = __ldg(ps + o + t + i * kRedThreads);
      uu[i] = __ldg(pu + o + t + i * kRedThreads);
      rr[i] = pr ? __ldg(pr + o + t + i * kRedThreads) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      msr_merge(m, s, r, mm[i], ss[i], rr[i]);
      u += uu[i];
    }
  }
  for (; t < n_tiles; t += kRedThreads) {
    msr_merge(m, s, r, __ldg(pm + o + t), __ldg(ps + o + t), pr ? __ldg(pr + o + t) : 0.f);
    u += __ldg(pu + o + t);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, off);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, off);
    const float r2 = __shfl_xor_sync(0xffffffffu, r, off);
    const float u2 = __shfl_xor_sync(0xffffffffu, u, off);
    msr_merge(m, s, r, m2, s2, r2);
    u += u2;
  }
  __shared__ float red[4][kRedThreads / 32];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { red[0][w] = m; red[1][w] = s; red[2][w] = u; red[3][w] = r; }
  __syncthreads();
  if (threadIdx.x == 0) {
    m = red[0][0]; s = red[1][0]; u = red[2][0]; r = red[3][0];
    for (int i = 1; i < kRedThreads / 32; ++i) {
      msr_merge(m, s, r, red[0][i], red[1][i], red[3][i]);
      u += red[2][i];
    }
    msu[row * kMsu + 0] = m;
    msu[row * kMsu + 1] = s;
    msu[row * kMsu + 2] = u;
    msu[row * kMsu + 3] = r;
  }
}

__global__ void __launch_bounds__(256) k_row_combine(const float* __restrict__ msu_all, int P, int64_t M,
                                                     const float* __restrict__ row_H, const float* __restrict__ row_w,
                                                     const uint8_t* __restrict__ row_class, float* __restrict__ row_lse,
                                                     float* __restrict__ row_loss, float* __restrict__ block_partials,
                                                     RowF2 f2) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
  float wl = 0.f;
  if (row < M) {
    float m = -INFINITY, s = 0.f, u = 0.f, r = 0.f;
    for (int p = 0; p < P; ++p) {
      const float* q = msu_all + (static_cast<int64_t>(p) * M + row) * kMsu;
      msr_merge(m, s, r, q[0], q[1], q[3]);
      u += q[2];
    }
    const float lse = m + logf(s);
    const uint8_t cls = row_class[row];
    float l = 0.f;
    if (cls == AURORA_ROW_ACCEPT && f2.rkl) {
      const float eqzt = r / s;  // E_q[z - t]
      l = eqzt - lse + f2.row_lse_t[row] + f2.beta * lse - u;
      f2.row_aux[row] = eqzt;
    } else if (cls == AURORA_ROW_DISCARD && f2.restricted) {
      // SPEC's restricted softmax: l = KL(p~ || q~) = H~ - u + lse_S with lse_S the
      // log-sum-exp of the support logits the staged forward kept
      const float* zr = f2.sup_z + row * f2.k_max;
      const int32_t* ir = f2.sup_idx + row * f2.k_max;
      float zm = -INFINITY;
      for (int j = 0; j < f2.k_max; ++j)
        if (ir[j] != INT32_MAX) zm = fmaxf(zm, zr[j]);
      float se = 0.f;
      for (int j = 0; j < f2.k_max; ++j)
        if (ir[j] != INT32_MAX) se += __expf(zr[j] - zm);
      const float lse_s = zm + logf(se);
      f2.row_aux[row] = lse_s;
      l = lse_s - u + row_H[row];
    } else if (cls != AURORA_ROW_PAD) {
      l = lse - u + row_H[row];
    }
    row_lse[row] = lse;
    if (row_loss) row_loss[row] = l;
    wl = row_w[row] * l;
  }
  // deterministic block tree reduction
  __shared__ float red[256];
  red[threadIdx.x] = wl;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) block_partials[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(256) k_loss_sum(const float* __restrict__ bp, int nb, float* __restrict__ loss) {
  __shared__ float red[256];
  float acc = 0.f;
  for (int i = threadIdx.x; i < nb; i += 256) acc += bp[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) loss[0] = red[0];
}

__global__ void __launch_bounds__(256) k_splitk_reduce(const float* __restrict__ part, int splits, int64_t n4,
                                                       float* __restrict__ out, int accumulate) {
  const int64_t stride = n4;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * 256) {
    float4 a = accumulate ? reinterpret_cast<const float4*>(out)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < splits; ++s) {
      const float4 b = __ldg(reinterpret_cast<const float4*>(part) + s * stride + i);
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    }
    reinterpret_cast<float4*>(out)[i] = a;
  }
}

// Test hook: full dz rows (SIMT, fp32 dot products from bf16).
__global__ void k_debug_dlogits(const __nv_bfloat16* __restrict__ H, const __nv_bfloat16* __restrict__ W, int64_t d,
                                int64_t V_local, int64_t vocab_offset, aurora_labels_t lab, const float* row_lse,
                                const float* dloss, const int32_t* rows, float* out) {
  const int r = blockIdx.y;
  const int64_t m = rows[r];
  const float g = dloss ? dloss[0] : 1.f;
  const float coef = g * lab.row_w[m];
  const float lse = row_lse[m];
  for (int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < V_local;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float z = 0.f;
    for (int64_t k = 0; k < d; ++k)
      z += __bfloat162float(H[m * d + k]) * __bfloat162float(W[v * d + k]);
    float dz = coef * expf(z - lse);
    for (int j = 0; j < lab.k_max; ++j)
      if (static_cast<int64_t>(lab.sup_idx[m * lab.k_max + j]) == v + vocab_offset)
        dz -= coef * lab.sup_p[m * lab.k_max + j];
    out[r * V_local + v] = dz;
  }
}

constexpr int kRsRows = 1024;  // dZ^T columns (rows m) per rescale CTA
__global__ void __launch_bounds__(256) k_dz_rescale(__nv_bfloat16* __restrict__ dzT, int64_t ld, int64_t M,
                                                    int64_t V_local, int bn, const float* __restrict__ pm,
                                                    int pm_stride, const float* __restrict__ row_lse,
                                                    const float* __restrict__ row_w, const float* __restrict__ dloss,
                                                    const uint8_t* __restrict__ row_class, int restricted) {
  __shared__ float F[kRsRows];
  const int h = blockIdx.x;  // tile half: tile h / 2, columns [0, 128) or [128, bn)
  const int64_t c0 = static_cast<int64_t>(h >> 1) * bn + ((h & 1) ? BN / 2 : 0);
  const int64_t c1 = min(static_cast<int64_t>(h >> 1) * bn + ((h & 1) ? bn : BN / 2), V_local);
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * kRsRows;
  const int64_t m1 = min(m0 + kRsRows, ld);
  const float g = dloss ? __ldg(dloss) : 1.f;
  for (int i = threadIdx.x; i < kRsRows; i += blockDim.x) {
    const int64_t m = m0 + i;
    float f = 0.f;
    if (m < M) {
      const float w = __ldg(row_w + m);
      const float mh = __ldg(pm + m * pm_stride + h);
      // restricted-softmax DISCARD rows: no full-vocabulary term (dz lives on the support only)
      const bool off = restricted && row_class[m] == AURORA_ROW_DISCARD;
      if (w != 0.f && mh != -INFINITY && !off) f = g * w * __expf(mh - __ldg(row_lse + m));
    }
    F[i] = f;
  }
  __syncthreads();
  if (c0 >= c1) return;
  const int nv = static_cast<int>((m1 - m0) >> 3);  // 8-row vectors per dZ^T row (ld % 8 == 0), <= 128
  // thread = one 8-row vector slot vi (its 8 factors in registers) of every cstep-th dZ^T row of
  // the half tile (cstep = blockDim / nv); 4 rows per step in flight (no per-element index
  // arithmetic)
  if (nv <= 0) return;
  const int vi = threadIdx.x % nv;
  const int cs = threadIdx.x / nv, cstep = blockDim.x / nv;
  if (cs >= cstep) return;
  float fv[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) fv[e] = F[vi * 8 + e];
  auto scale8 = [&](uint4& x) {
    uint32_t* w = &x.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&w[e]);
      const float2 f = __bfloat1622float2(b);
      b = __floats2bfloat162_rn(f.x * fv[2 * e], f.y * fv[2 * e + 1]);
      w[e] = *reinterpret_cast<uint32_t*>(&b);
    }
  };
  uint4* base = reinterpret_cast<uint4*>(dzT + m0) + vi;
  const int64_t ldv = ld / 8;  // uint4 per dZ^T row
  int64_t c = c0 + cs;
  for (; c + 3 * cstep < c1; c += 4 * cstep) {
    uint4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = base[(c + u * cstep) * ldv];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      scale8(x[u]);
      base[(c + u * cstep) * ldv] = x[u];
    }
  }
  for (; c < c1; c += cstep) {
    uint4 x = base[c * ldv];
    scale8(x);
    base[c * ldv] = x;
  }
}

__global__ void k_dz_support_fix(__nv_bfloat16* __restrict__ dzT, int64_t ld, int64_t M, int64_t V_local,
                                 int64_t vocab_offset, const int32_t* __restrict__ sup_idx,
                                 const float* __restrict__ sup_p, const float* __restrict__ sup_z, int k_max,
                                 const float* __restrict__ row_lse, const float* __restrict__ row_w,
                                 const float* __restrict__ dloss, const uint8_t* __restrict__ row_class,
                                 const float* __restrict__ row_aux, int restricted) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= M * k_max) return;
  const int64_t m = i / k_max;
  const int32_t gid = sup_idx[i];
  if (gid == INT32_MAX) return;
  const int64_t loc = static_cast<int64_t>(gid) - vocab_offset;
  if (loc < 0 || loc >= V_local) return;
  const float coef = (dloss ? __ldg(dloss) : 1.f) * row_w[m];
  // restricted DISCARD rows: q~_j = exp(z_j - lse_S) over the support (lse_S from the combine)
  const float lse = (restricted && row_class[m] == AURORA_ROW_DISCARD) ? row_aux[m] : row_lse[m];
  dzT[loc * ld + m] = __float2bfloat16_rn(coef * (__expf(sup_z[i] - lse) - sup_p[i]));
}

cudaError_t launch_dz_rescale(__nv_bfloat16* dzT, int64_t ld, int64_t M, int64_t V_local, int bn, int n_tiles,
                              const float* pm, const float* row_lse, const float* row_w, const float* dloss,
                              const uint8_t* row_class, int restricted, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>(2 * n_tiles), static_cast<unsigned>((ld + kRsRows - 1) / kRsRows));
  k_dz_rescale<<<grid, 256, 0, s>>>(dzT, ld, M, V_local, bn, pm, 2 * n_tiles, row_lse, row_w, dloss, row_class,
                                    restricted);
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_dz_support_fix(__nv_bfloat16* dzT, int64_t ld, int64_t M, int64_t V_local, int64_t vocab_offset,
                                  const aurora_labels_t* lab, const float* sup_z, const float* row_lse,
                                  const float* dloss, int restricted, cudaStream_t s) {
  const int64_t n = M * lab->k_max;
  k_dz_support_fix<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
      dzT, ld, M, V_local, vocab_offset, lab->sup_idx, lab->sup_p, sup_z, lab->k_max, row_lse, lab->row_w, dloss,
      lab->row_class, lab->row_aux, restricted);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_reduce_partials(const float* pm, const float* ps, const float* pu, const float* pr, int64_t M,
                                   int n_tiles, float* msu, cudaStream_t s) {
  k_reduce_partials<<<static_cast<unsigned>(M), kRedThreads, 0, s>>>(pm, ps, pu, pr, M, n_tiles, msu);
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_row_combine(const float* msu_all, int P, int64_t M, const float* row_H, const float* row_w,
                               const uint8_t* row_class, float* row_lse, float* row_loss, float* block_partials,
                               int* nblocks_out, const RowF2& f2, cudaStream_t s) {
  const int nb = static_cast<int>((M + 255) / 256);
  k_row_combine<<<nb, 256, 0, s>>>(msu_all, P, M, row_H, row_w, row_class, row_lse, row_loss, block_partials, f2);
  count_launch();
  *nblocks_out = nb;
  return cudaGetLastError();
}
cudaError_t launch_loss_sum(const float* bp, int nb, float* loss, cudaStream_t s) {
  k_loss_sum<<<1, 256, 0, s>>>(bp, nb, loss);
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_splitk_reduce(const float* partials, int splits, int64_t n_elems, float* out, int accumulate,
                                 cudaStream_t s) {
  const int64_t n4 = n_elems / 4;
  int64_t blocks = (n4 + 255) / 256;
  if (blocks > 4 * kNumSMs) blocks = 4 * kNumSMs;
  k_splitk_reduce<<<static_cast<unsigned>(blocks), 256, 0, s>>>(partials, splits, n4, out, accumulate);
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_debug_dlogits(const __nv_bfloat16* H, const __nv_bfloat16* W, int64_t M, int64_t d,
                                 int64_t V_local, int64_t vocab_offset, const aurora_labels_t* lab,
                                 const float* row_lse, const float* dloss, const int32_t* rows, int n_rows,
                                 float* out, cudaStream_t s) {
  (void)M;
  dim3 grid(64, n_rows);
  k_debug_dlogits<<<grid, 256, 0, s>>>(H, W, d, V_local, vocab_offset, *lab, row_lse, dloss, rows, out);
  count_launch();
  return cudaGetLastError();
}

}  // namespace aur

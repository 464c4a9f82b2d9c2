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
constexpr int KM = AURORA_MAX_K;  // register list length (runtime k <= KM)

// (v, i) ranks before (w, j)?  value desc, index asc.
__device__ __forceinline__ bool better(float v, int32_t i, float w, int32_t j) {
  return v > w || (v == w && i < j);
}

struct TopList {
  float v[KM];
  int32_t i[KM];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int j = 0; j < KM; ++j) { v[j] = -INFINITY; i[j] = INT32_MAX; }
  }
  // bubble insertion keeping (value desc, index asc)
  __device__ __forceinline__ void insert(float cv, int32_t ci) {
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      const bool sw = better(cv, ci, v[j], i[j]);
      const float tv = v[j];
      const int32_t ti = i[j];
      v[j] = sw ? cv : tv;
      i[j] = sw ? ci : ti;
      cv = sw ? tv : cv;
      ci = sw ? ti : ci;
    }
  }
  __device__ __forceinline__ float kth(int k) const {
    float t = v[0];
#pragma unroll
    for (int j = 0; j < KM; ++j) t = (j == k - 1) ? v[j] : t;
    return t;
  }
  __device__ __forceinline__ int32_t kth_idx(int k) const {
    int32_t t = i[0];
#pragma unroll
    for (int j = 0; j < KM; ++j) t = (j == k - 1) ? i[j] : t;
    return t;
  }
  __device__ __forceinline__ void pop_front() {
#pragma unroll
    for (int j = 0; j < KM - 1; ++j) { v[j] = v[j + 1]; i[j] = i[j + 1]; }
    v[KM - 1] = -INFINITY;
    i[KM - 1] = INT32_MAX;
  }
};

// Warp-wide k-way merge of per-lane sorted lists; after the call every lane holds
// the merged top-k in (ov, oi)[0..k).
__device__ __forceinline__ void warp_merge(TopList& L, int k, float* ov, int32_t* oi) {
  for (int r = 0; r < k; ++r) {
    float bv = L.v[0];
    int32_t bi = L.i[0];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float ov2 = __shfl_xor_sync(0xffffffffu, bv, off);
      const int32_t oi2 = __shfl_xor_sync(0xffffffffu, bi, off);
      if (better(ov2, oi2, bv, bi)) { bv = ov2; bi = oi2; }
    }
    ov[r] = bv;
    oi[r] = bi;
    if (L.i[0] == bi && L.v[0] == bv && bi != INT32_MAX) L.pop_front();
  }
}

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
}  // namespace

// --------------------------------------------------------------------------- A2 scan
// grid (M * nseg), 256 threads.  Segment [seg*seg_len, min(V_local, +seg_len)).
__global__ void __launch_bounds__(256) k_target_scan(VerifyLaunch p) {
  const int row = blockIdx.x / p.nseg;
  const int seg = blockIdx.x % p.nseg;
  const int k = p.k_max;
  const int64_t c0 = static_cast<int64_t>(seg) * p.seg_len;
  const int64_t c1 = min(p.V_local, c0 + p.seg_len);
  const uint16_t* T = p.T + static_cast<int64_t>(row) * p.ldT;
  TopList L;
  L.init();
  float thr = -INFINITY;
  uint32_t bad = 0;

  auto consider = [&](float v, int64_t col) {
    if (v > thr) {  // later columns of this thread can only lose ties (index asc)
      L.insert(v, static_cast<int32_t>(col));
      thr = L.kth(k);
    }
  };

  const bool aligned = ((reinterpret_cast<uintptr_t>(T + c0) & 15) == 0);
  if (aligned) {
    const int64_t nvec = (c1 - c0) >> 3;
    const uint4* src = reinterpret_cast<const uint4*>(T + c0);
    constexpr int U = 8;
    int64_t it = threadIdx.x;
    for (; it + (U - 1) * 256 < nvec; it += U * 256) {
      uint4 w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint4* a = src + it + u * 256;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(w[u].x), "=r"(w[u].y), "=r"(w[u].z), "=r"(w[u].w)
                     : "l"(a));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        // non-finite: any |x| exponent all-ones
        const uint32_t ax = __vmaxu2(__vmaxu2(w[u].x & 0x7FFF7FFFu, w[u].y & 0x7FFF7FFFu),
                                     __vmaxu2(w[u].z & 0x7FFF7FFFu, w[u].w & 0x7FFF7FFFu));
        bad |= ((ax & 0xFFFFu) >= 0x7F80u) | ((ax >> 16) >= 0x7F80u);
        const __nv_bfloat162 m2 = __hmax2(__hmax2(*reinterpret_cast<const __nv_bfloat162*>(&w[u].x),
                                                  *reinterpret_cast<const __nv_bfloat162*>(&w[u].y)),
                                          __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&w[u].z),
                                                  *reinterpret_cast<const __nv_bfloat162*>(&w[u].w)));
        const float gm = fmaxf(__low2float(m2), __high2float(m2));
        if (gm > thr) {
          const int64_t col = c0 + (it + u * 256) * 8;
          const uint32_t ws[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            consider(bf16_lo(ws[e]), col + 2 * e);
            consider(bf16_hi(ws[e]), col + 2 * e + 1);
          }
        }
      }
    }
    for (; it < nvec; it += 256) {
      const uint4 w = src[it];
      const int64_t col = c0 + it * 8;
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t a = ws[e] & 0x7FFF7FFFu;
        bad |= ((a & 0xFFFFu) >= 0x7F80u) | ((a >> 16) >= 0x7F80u);
        consider(bf16_lo(ws[e]), col + 2 * e);
        consider(bf16_hi(ws[e]), col + 2 * e + 1);
      }
    }
    for (int64_t col = c0 + nvec * 8 + threadIdx.x; col < c1; col += 256) {
      const uint32_t b = T[col];
      bad |= ((b & 0x7FFFu) >= 0x7F80u);
      consider(__uint_as_float(b << 16), col);
    }
  } else {
    for (int64_t col = c0 + threadIdx.x; col < c1; col += 256) {
      const uint32_t b = T[col];
      bad |= ((b & 0x7FFFu) >= 0x7F80u);
      consider(__uint_as_float(b << 16), col);
    }
  }
  if (bad) atomicOr(p.lab.status, AURORA_STATUS_NONFINITE);

  // ---- block merge: per warp, then across the 8 warps
  __shared__ float s_v[8][KM];
  __shared__ int32_t s_i[8][KM];
  float ov[KM];
  int32_t oi[KM];
  warp_merge(L, k, ov, oi);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    for (int j = 0; j < k; ++j) { s_v[warp][j] = ov[j]; s_i[warp][j] = oi[j]; }
  }
  __syncthreads();
  if (warp == 0) {
    TopList L2;
    L2.init();
    if (lane < 8) {
      for (int j = 0; j < k; ++j) { L2.v[j] = s_v[lane][j]; L2.i[j] = s_i[lane][j]; }
    }
    warp_merge(L2, k, ov, oi);
    if (lane == 0) {
      const int64_t o = (static_cast<int64_t>(row) * p.nseg + seg) * k;
      for (int j = 0; j < k; ++j) {
        p.cand_val[o + j] = ov[j];
        p.cand_idx[o + j] = (oi[j] == INT32_MAX) ? INT32_MAX : static_cast<int32_t>(oi[j] + p.vocab_offset);
      }
    }
  }
}

// --------------------------------------------------------------------------- A2 merge
// warp per row: merge `nlists` (<= 32) sorted lists of length k -> top list + argmax.
__global__ void __launch_bounds__(256) k_topk_merge(VerifyLaunch p, const float* in_val, const int32_t* in_idx,
                                                    int nlists, int64_t row_stride, int64_t list_stride) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= p.M) return;
  const int k = p.k_max;
  TopList L;
  L.init();
  if (lane < nlists) {
    const int64_t o = static_cast<int64_t>(row) * row_stride + lane * list_stride;
    for (int j = 0; j < k; ++j) { L.v[j] = in_val[o + j]; L.i[j] = in_idx[o + j]; }
  }
  float ov[KM];
  int32_t oi[KM];
  warp_merge(L, k, ov, oi);
  if (lane == 0) {
    for (int j = 0; j < k; ++j) {
      p.top_val[static_cast<int64_t>(row) * k + j] = ov[j];
      p.top_idx[static_cast<int64_t>(row) * k + j] = oi[j];
    }
    p.lab.target_argmax[row] = oi[0];
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
// thread per row.
__global__ void __launch_bounds__(256) k_finalize(VerifyLaunch p) {
  const int64_t m = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
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
  float v[KM];
  int32_t ix[KM];
  const float* tv = p.top_val + m * km;
  const int32_t* ti = p.top_idx + m * km;
  float esum = 0.f;
  const float t0 = k > 0 ? tv[0] : 0.f;
  for (int j = 0; j < k; ++j) {
    v[j] = tv[j] - t0;  // <= 0
    ix[j] = ti[j];
    esum += expf(v[j]);
  }
  const float lz = logf(esum);
  float H = 0.f;
  for (int j = 0; j < k; ++j) {
    const float lp = v[j] - lz;
    v[j] = expf(lp);  // p~
    H += v[j] * lp;
  }
  if (k == 1) H = 0.f;
  // sort support by global index (insertion sort, k <= 16)
  for (int a = 1; a < k; ++a) {
    const float pv = v[a];
    const int32_t pi = ix[a];
    int b = a - 1;
    while (b >= 0 && ix[b] > pi) { v[b + 1] = v[b]; ix[b + 1] = ix[b]; --b; }
    v[b + 1] = pv;
    ix[b + 1] = pi;
  }
  for (int j = 0; j < km; ++j) {
    p.lab.sup_idx[m * km + j] = j < k ? ix[j] : INT32_MAX;
    p.lab.sup_p[m * km + j] = j < k ? v[j] : 0.f;
  }
  p.lab.row_H[m] = H;
  p.lab.row_w[m] = w;
}

// --------------------------------------------------------------------------- launchers
cudaError_t launch_target_scan(const VerifyLaunch& p, cudaStream_t s) {
  k_target_scan<<<static_cast<unsigned>(p.M) * p.nseg, 256, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_topk_merge(const VerifyLaunch& p, const float* in_val, const int32_t* in_idx, int nlists,
                              int64_t row_stride, int64_t list_stride, cudaStream_t s) {
  k_topk_merge<<<(p.M + 7) / 8, 256, 0, s>>>(p, in_val, in_idx, nlists, row_stride, list_stride);
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_verify(const VerifyLaunch& p, cudaStream_t s) {
  k_verify<<<(p.R + 7) / 8, 256, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_finalize(const VerifyLaunch& p, cudaStream_t s) {
  k_finalize<<<(p.M + 255) / 256, 256, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace aur

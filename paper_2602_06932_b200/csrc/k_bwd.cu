// k_bwd.cu — the whole backward as ONE persistent tcgen05 kernel.
//
// The three contractions of the lm_head backward reduce over different dimensions
// (dz recompute over d, dW over the rows M, dH over the vocabulary), so the bf16 dLogits
// are staged per vocab chunk (1/8 of V_local, double-buffered => at most 1/4 of the
// local [M x V_local] dLogits is ever live).  Instead of 3 launches per chunk (each with
// its own wave-quantisation tail, and dW's HBM-bound stores never overlapping the
// tensor-bound tiles), one launch walks a unified tile queue
//
//     DZ(0) | DZ(1) | DH(0) | DW(0) | DZ(2) | DH(1) | DW(1) | ... | DH(n-1) | DW(n-1)
//
// claimed dynamically (atomicAdd) by 148 persistent CTAs, with cross-CTA dependency
// counters in global memory:
//   * DH(c)/DW(c) tiles read dZ^T[c & 1]: their producer waits dz_done[c] == #DZ(c).
//   * DZ(c) (c >= 2) overwrites buffer c & 1: its epilogue waits rd_done[c-2] ==
//     #DH(c-2) + #DW(c-2) before the first store.
//   * DH(c) tile (m, n, split) accumulates onto the same output as DH(c-1): its epilogue
//     waits dh_flag == c, so the fp32 sums happen in chunk order (deterministic).
// Every dependency points to a tile that was claimed EARLIER in the queue, so it is
// already owned by a running CTA whose earlier work never waits on later tiles: no
// deadlock.  Stores: dz via st.global (dZ^T, coalesced over rows), dW / dH via TMA bulk
// tensor stores / reduce-adds from 64B-swizzled smem staging.
#include "gemm_dev.cuh"

namespace aur {

namespace {
__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void spin_geq(const int32_t* p, int target) {
  while (ld_acquire(p) < target) __nanosleep(128);
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory"); }

struct Unit {
  int type, chunk, mt, nt, sp, kb0, kb1;
};
__device__ __forceinline__ Unit decode(const BwdArgs& a, int u) {
  int s = 0;
  while (s + 1 < a.nseg && u >= a.seg[s + 1].base) ++s;
  const BwdSeg& g = a.seg[s];
  const int i = u - g.base;
  Unit x;
  x.type = g.type;
  x.chunk = g.chunk;
  if (g.type == BT_DW) {  // n-fastest: the dZ^T rows of a vocab tile are reused from L2
    x.nt = i % g.n_tiles;
    x.mt = i / g.n_tiles;
    x.sp = 0;
  } else {
    x.mt = i % g.m_tiles;
    const int r = i / g.m_tiles;
    x.nt = r % g.n_tiles;
    x.sp = r / g.n_tiles;
  }
  x.kb0 = x.sp * g.kb_per_split;
  x.kb1 = min(g.kb_total, x.kb0 + g.kb_per_split);
  return x;
}
}  // namespace

__global__ void __launch_bounds__(kGemmThreads, 1)
    k_bwd_fused(const __grid_constant__ BwdMaps maps, const __grid_constant__ BwdArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kSmemA;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sB + kStages * kSmemB);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* sfull_bar = tempty_bar + 2;
  uint64_t* sempty_bar = sfull_bar + kSchedDepth;
  int32_t* s_sched = reinterpret_cast<int32_t*>(sempty_bar + kSchedDepth);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(s_sched + kSchedDepth);
  uint8_t* stage = smem + kStages * (kSmemA + kSmemB) + 1024;  // 1024-B aligned staging

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&maps.H_k);
    tma_prefetch_desc(&maps.W_k);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], kEpiWarps);
    }
    for (int d = 0; d < kSchedDepth; ++d) {
      mbar_init(&sfull_bar[d], 1);
      mbar_init(&sempty_bar[d], 1 + kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int units = args.total_units;

  auto consumer_next = [&](uint32_t& slot, uint32_t& ph, bool is_mma) -> int {
    mbar_wait(&sfull_bar[slot], ph);
    const int u = *reinterpret_cast<volatile int32_t*>(&s_sched[slot]);
    if (is_mma) {
      mbar_arrive(&sempty_bar[slot]);
    } else {
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty_bar[slot]);
    }
    if (++slot == kSchedDepth) { slot = 0; ph ^= 1; }
    return u;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t st = 0, phase = 0, sslot = 0, sph = 0;
      for (;;) {
        const int u = atomicAdd(args.tile_counter, 1);
        mbar_wait(&sempty_bar[sslot], sph ^ 1);
        s_sched[sslot] = u;
        mbar_arrive(&sfull_bar[sslot]);
        if (++sslot == kSchedDepth) { sslot = 0; sph ^= 1; }
        if (u >= units) break;
        const Unit x = decode(args, u);
        const int b = x.chunk & 1;
        if (x.type != BT_DZ) {  // dZ^T[b] of this chunk must be complete (written by other CTAs)
          spin_geq(args.dz_done + x.chunk, args.n_dz[x.chunk]);
          fence_proxy_async_global();
        }
        const int32_t c0 = static_cast<int32_t>(args.c0[x.chunk]);
        for (int kb = x.kb0; kb < x.kb1; ++kb) {
          mbar_wait(&empty_bar[st], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[st], kSmemA + kSmemB);
          uint8_t* a = sA + st * kSmemA;
          uint8_t* bb = sB + st * kSmemB;
          if (x.type == BT_DZ) {  // Z^T tile = H[rows] . W[vocab]^T, K = d
            tma_load_2d(&maps.H_k, &full_bar[st], a, kb * BK, x.mt * BM);
            tma_load_2d(&maps.W_k, &full_bar[st], bb, kb * BK, c0 + x.nt * BN);
          } else if (x.type == BT_DW) {  // dW[vocab, d] = dZ^T[vocab, m] . H[m, d], K = M
            tma_load_2d(&maps.Z_k[b], &full_bar[st], a, kb * BK, x.mt * BM);
#pragma unroll
            for (int i = 0; i < BN / 64; ++i)
              tma_load_2d(&maps.H_mn, &full_bar[st], bb + i * (BK * 128), x.nt * BN + i * 64, kb * BK);
          } else {  // dH[m, d] += dZ[m, vocab] . W[vocab, d], K = vocab chunk
#pragma unroll
            for (int i = 0; i < BM / 64; ++i)
              tma_load_2d(&maps.Z_mn[b], &full_bar[st], a + i * (BK * 128), x.mt * BM + i * 64, kb * BK);
#pragma unroll
            for (int i = 0; i < BN / 64; ++i)
              tma_load_2d(&maps.W_mn, &full_bar[st], bb + i * (BK * 128), x.nt * BN + i * 64, c0 + kb * BK);
          }
          if (++st == kStages) { st = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      uint32_t st = 0, phase = 0, acc = 0, acc_phase = 0, sslot = 0, sph = 0;
      for (;;) {
        const int u = consumer_next(sslot, sph, true);
        if (u >= units) break;
        const Unit x = decode(args, u);
        const bool a_mn = (x.type == BT_DH);
        const bool b_mn = (x.type != BT_DZ);
        const uint32_t idesc = umma_idesc_bf16(BM, BN, a_mn, b_mn);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = x.kb0; kb < x.kb1; ++kb) {  // (empty split: commit with no MMA)
          mbar_wait(&full_bar[st], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + st * kSmemA);
          const uint32_t b_base = smem_u32(sB + st * kSmemB);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16(d_tmem, operand_desc_rt(a_base, k, a_mn), operand_desc_rt(b_base, k, b_mn), idesc,
                      (kb > x.kb0 || k > 0) ? 1u : 0u);
          umma_commit(&empty_bar[st]);
          if (++st == kStages) { st = 0; phase ^= 1; }
        }
        umma_commit(&tfull_bar[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (8 warps)
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int cbeg = half * (BN / 2);
    const bool leader = (threadIdx.x == 64);
    uint8_t* slots = stage + (warp - 2) * (2 * 2048);
    uint32_t epi_chunk = 0, acc = 0, acc_phase = 0, sslot = 0, sph = 0;
    for (;;) {
      const int u = consumer_next(sslot, sph, false);
      if (u >= units) break;
      const Unit x = decode(args, u);
      const int c = x.chunk;
      const int64_t vc = args.vc[c];
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);

      if (x.type == BT_DZ) {
        // ---- dz = g w (exp(z - lse) - p~) -> bf16 dZ^T[buffer c&1]
        if (c >= 2) {
          if (leader) spin_geq(args.rd_done + (c - 2), args.n_rd[c - 2]);
          epi_bar();
        }
        const int64_t row = static_cast<int64_t>(x.mt) * BM + q * 32 + lane;
        const bool row_ok = row < args.M;
        const int64_t col0 = static_cast<int64_t>(x.nt) * BN;  // local column within the chunk
        const int64_t rem = vc - col0;
        const int ncols = rem < BN ? static_cast<int>(rem) : BN;
        // columns [ncols, round_up(ncols, 64)) are stored as zeros: the dH tiles read the
        // buffer in whole 64-row k-blocks and must not pick up a previous chunk's values
        const int npad = (ncols + 63) & ~63;
        const int cend = npad < cbeg + BN / 2 ? npad : cbeg + BN / 2;
        SupCursor cur;
        cur.idx = args.sup_idx + (row_ok ? row : 0) * args.k_max;
        cur.p = args.sup_p + (row_ok ? row : 0) * args.k_max;
        cur.k = row_ok ? args.k_max : 0;
        cur.limit = vc;
        cur.gid0 = args.vocab_offset + args.c0[c];
        cur.seek(col0 + cbeg);
        float coef = 0.f, lse2 = 0.f;
        if (row_ok) {
          const float g = args.dloss ? __ldg(args.dloss) : 1.f;
          coef = g * __ldg(args.row_w + row);
          lse2 = __ldg(args.row_lse + row) * kLog2e;
        }
        __nv_bfloat16* dzT = args.dzT[c & 1];
        for (int cb = cbeg; cb < cend; cb += 32) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(taddr + cb, r);
          tmem_ld_wait();
          float z[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) z[j] = coef * ex2_approx(fmaf(__uint_as_float(r[j]), kLog2e, -lse2));
          while (cur.nxt < col0 + cb + 32) {
            const int jj = static_cast<int>(cur.nxt - col0 - cb);
            const float sub = coef * cur.nxt_p;
#pragma unroll
            for (int j = 0; j < 32; ++j) z[j] = (j == jj) ? z[j] - sub : z[j];
            cur.advance();
          }
          if (row_ok) {
            __nv_bfloat16* dst = dzT + (col0 + cb) * args.ld_dzT + row;
            const int nj = (cb + 32 <= npad) ? 32 : npad - cb;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < nj) dst[j * args.ld_dzT] = __float2bfloat16_rn(cb + j < ncols ? z[j] : 0.f);
          }
        }
        __threadfence();
        fence_proxy_async_global();  // generic-proxy stores -> later async-proxy (TMA) reads
        epi_bar();
        if (leader) atomicAdd(args.dz_done + c, 1);
      } else {
        // ---- dW / dH tile: TMEM -> swizzled smem -> TMA bulk store / reduce-add
        const bool is_dh = (x.type == BT_DH);
        // The tile's MMAs are complete (tfull), i.e. its reads of dZ^T[c & 1] are done:
        // release the buffer for DZ(c + 2) before doing the stores.
        if (leader) {
          __threadfence();
          atomicAdd(args.rd_done + c, 1);
        }
        int32_t* flag = nullptr;
        if (is_dh) {
          flag = args.dh_flag + (static_cast<int64_t>(x.sp) * args.dh_n_tiles + x.nt) * args.dh_m_tiles + x.mt;
          if (c > 0) {
            if (leader) spin_geq(flag, c);
            epi_bar();
          }
        }
        const bool accumulate = is_dh ? (c > 0) : (args.accumulate_dW != 0);
        const CUtensorMap* out = is_dh ? &maps.O_H : &maps.O_W;
        const int32_t ybase = is_dh ? (x.mt * BM + q * 32)
                                    : static_cast<int32_t>(args.c0[c] + static_cast<int64_t>(x.mt) * BM + q * 32);
        const int32_t zc = is_dh ? x.sp : 0;
        const int64_t ncols_n = args.d - static_cast<int64_t>(x.nt) * BN;
        const int ncols = ncols_n < BN ? static_cast<int>(ncols_n) : BN;
        const int cend = ncols < cbeg + BN / 2 ? ncols : cbeg + BN / 2;
        const bool empty = x.kb0 >= x.kb1;  // split with no k-blocks: contributes zeros
        for (int cb = cbeg; cb < cend; cb += 16) {
          uint32_t r[16];
          tmem_ld_32x32b_x16(taddr + cb, r);
          uint8_t* slot = slots + (epi_chunk & 1) * 2048;
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
          tmem_ld_wait();
          // chunk widths are multiples of 256 except the last chunk, which ends at V_local
          // (clipped by the map): a box never spills into the next chunk's rows.
          const bool mine = !empty;
          const uint32_t sbase = smem_u32(slot) + lane * 64;
          const uint32_t sw = (lane >> 1) & 3;
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
            sts128(sbase + ((cc ^ sw) << 4), mine ? __uint_as_float(r[4 * cc]) : 0.f,
                   mine ? __uint_as_float(r[4 * cc + 1]) : 0.f, mine ? __uint_as_float(r[4 * cc + 2]) : 0.f,
                   mine ? __uint_as_float(r[4 * cc + 3]) : 0.f);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && !(empty && accumulate)) {
            const int32_t xx = x.nt * BN + cb;
            if (accumulate) tma_reduce_add_3d(out, slot, xx, ybase, zc);
            else tma_store_3d(out, slot, xx, ybase, zc);
            bulk_commit();
          }
          ++epi_chunk;
        }
        // dH: the next chunk's reduce-add onto this tile must see these sums (ordered,
        // deterministic fp32 accumulation): wait for the bulk ops, then publish the flag.
        if (is_dh && c + 1 < args.nchunks) {
          if (lane == 0) bulk_wait<0>();
          fence_proxy_async_all();
          __threadfence();
          epi_bar();
          if (leader) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(c + 1) : "memory");
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (lane == 0) bulk_wait<0>();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

cudaError_t launch_bwd_fused(const BwdMaps& maps, const BwdArgs& args, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_bwd_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmSmem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (args.total_units <= 0) return cudaSuccess;
  const int grid = args.total_units < kNumSMs ? args.total_units : kNumSMs;
  k_bwd_fused<<<grid, kGemmThreads, kGemmSmem, s>>>(maps, args);
  count_launch();
  return cudaGetLastError();
}

}  // namespace aur

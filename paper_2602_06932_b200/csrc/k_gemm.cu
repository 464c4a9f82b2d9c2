// k_gemm.cu — persistent warp-specialised tcgen05 GEMM engine for the lm_head phases.
//
// One CTA per SM (320 threads):
//   warp 0      TMA producer: 4-stage ring of {A 128x64, B 256x64} bf16 tiles, SW128
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=256, K=16)
//   warps 2..9  epilogue: tcgen05.ld 32x32b (warp w reads TMEM lanes 32*(w%4)..; two warps
//               per lane quadrant split the 256 columns)
// Two 128x256 fp32 accumulators (512 TMEM columns) let the epilogue of tile i overlap
// the MMAs of tile i+1.  Tiles are visited m-fastest, so all row tiles of one vocab
// tile run back to back and W (the large operand) is streamed from HBM once per phase.
//
// Epilogues (the fused hot ops of SURVEY §8(a)):
//   EPI_FWD_STATS  A5: per (row, vocab tile) running max m, sum exp(z-m) and the
//                  support dot u = sum_{j in S} p~_j z_j  (Eq. 3).
//                  Z never leaves TMEM.
//   EPI_BWD_DZ     A7: dz = g w (exp(z - lse) - p~) (gradient of KL(p~||q)),
//                  rounded to bf16 and stored TRANSPOSED into the chunk workspace
//                  dZ^T[v, m] (coalesced: a warp store covers 32 consecutive rows).
//   EPI_STORE_F32  A8/A9: fp32 tile store (overwrite / accumulate / split-K slot).
//   EPI_FWD_STAGE  A5 plus the staged half of A7 (default Eq. 3 path): the statistics of
//                  EPI_FWD_STATS with an exact per-(row, tile half) max, and the softmax
//                  numerators exp(z - m_half) stored as bf16 into the dZ^T workspace, so
//                  the backward needs no recompute GEMM (k_dz_rescale finishes dz).
#include <cfloat>
#include <climits>

#include "gemm_dev.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace aur {

int g_pair_max_clusters = -1;

// PAIR = 1: one CTA per 128x256 tile (tcgen05.mma.cta_group::1, M = 128).
// PAIR = 2: a 2-CTA cluster per 256x256 tile (tcgen05.mma.cta_group::2, M = 256): each
//   CTA TMA-loads its own 128 rows of A and HALF of B (128 of the 256 columns) into its
//   own smem, crediting the leader's full barrier; the leader issues the pair MMA and
//   commits to both CTAs' barriers; each CTA's TMEM holds its 128 rows x 256 columns and
//   its epilogue releases the leader's TMEM-empty barrier.  Operand traffic per flop
//   drops by a third and the stage ring grows from 4 x 48 KB to 6 x 32 KB.
//
// TBN: tile width (vocab columns per tile).  256 by default; 224 / 192 for K-major B with
// single-CTA tiles, chosen by the host when the narrower tile fills the 148 SMs' waves
// better (e.g. M = 384 rows x a 32K-column dz chunk: 378 tiles = 2.55 waves at 256 wide,
// 432 tiles = 2.92 waves at 224).  Accumulators stay at TMEM columns 0 / 256.
// F2: the 32 bf16 target logits T[row, c .. c+32) as floats (n valid; rest -inf).
__device__ __forceinline__ void load_t32(const uint16_t* trow, int64_t c, int n, int vec, float* t) {
  if (vec && n == 32) {
    const uint4* p = reinterpret_cast<const uint4*>(trow + c);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 w = __ldg(p + i);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        t[8 * i + 2 * e] = __uint_as_float(ws[e] << 16);
        t[8 * i + 2 * e + 1] = __uint_as_float(ws[e] & 0xFFFF0000u);
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) t[j] = j < n ? __uint_as_float(static_cast<uint32_t>(__ldg(trow + c + j)) << 16) : -INFINITY;
  }
}

// Shared-memory plan of one instantiation.  The fp32 store epilogue keeps kSlots 2 KB
// bulk-store slots per epilogue warp (measured: 6 slots instead of 2, 32x32 boxes, or
// half the warps on LSU stores do not raise the store-bound rate, and fewer ring stages
// slow K = 384).
template <int EPI, bool A_MN, int PAIR, int TBN>
struct SmemPlan {
  static constexpr int kSB = (TBN / PAIR) * BK * 2;  // B bytes per stage in this CTA
  static constexpr int kStageBytes = kSmemA + kSB;
  static constexpr bool kStore = EPI == EPI_STORE_F32 || EPI == EPI_STORE_BF16;
  static constexpr int kSt = PAIR == 2 ? 6 : kStages;
  static constexpr int kRing = kSt * kStageBytes;
  static constexpr int kSlots = kStore ? 2 : 0;  // 2 KB bulk-store slots per warp
  static constexpr int kStaging = kEpiWarps * kSlots * 2048;
  static constexpr int kBytes = kRing + 1024 /*barriers*/ + 1024 /*base alignment*/ + kStaging;
  static_assert(kBytes <= 232448, "dynamic smem per CTA");
  static_assert(kSt * kStageBytes <= kStages * (kSmemA + kSmemB), "ring");
  static_assert(!kStore || kSlots * 2048 >= 32 * kStgLd * 4, "LSU staging fits a warp's slots");
};

template <int EPI, bool A_MN, bool B_MN, int PAIR, int TBN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_umma_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC, const GemmArgs args) {
  using Plan = SmemPlan<EPI, A_MN, PAIR, TBN>;
  constexpr bool kStage = EPI == EPI_FWD_STAGE;
  constexpr bool kFwd = EPI == EPI_FWD_STATS || EPI == EPI_FWD_STATS_T || kStage;
  constexpr bool kDz = EPI == EPI_BWD_DZ || EPI == EPI_BWD_DZ_T;
  constexpr bool kT = EPI == EPI_FWD_STATS_T || EPI == EPI_BWD_DZ_T;
  static_assert(TBN == BN || (PAIR == 1 && !B_MN), "narrow tiles: single-CTA, K-major B only");
  static_assert(TBN % 32 == 0 && TBN > BN / 2 && TBN <= BN, "tile width");
  constexpr int kSt = Plan::kSt;
  constexpr int kSB = Plan::kSB;
  constexpr int kStageBytes = Plan::kStageBytes;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kSt * kSmemA;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Plan::kRing);
  uint64_t* empty_bar = full_bar + kSt;
  uint64_t* tfull_bar = empty_bar + kSt;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* sfull_bar = tempty_bar + 2;        // tile-index ring (dynamic scheduler)
  uint64_t* sempty_bar = sfull_bar + kSchedDepth;
  int32_t* s_sched = reinterpret_cast<int32_t*>(sempty_bar + kSchedDepth);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(s_sched + kSchedDepth);
  // epilogue staging, 1024-B aligned (the 64B / 128B swizzle patterns repeat every 512 / 1024 B)
  float* stage_f32 = reinterpret_cast<float*>(smem + Plan::kRing + 1024);
  static_assert((2 * kSt + 4 + 2 * kSchedDepth) * 8 + 4 * kSchedDepth + 4 <= 1024, "barrier area");

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = (PAIR == 2) ? cluster_ctarank() : 0u;  // 0 = pair leader

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if ((EPI == EPI_STORE_F32 && args.tma_store) || EPI == EPI_STORE_BF16) tma_prefetch_desc(&tmC);
    for (int s = 0; s < kSt; ++s) {
      mbar_init(&full_bar[s], PAIR);  // leader: own expect_tx arrive + peer's remote arrive
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], PAIR * kEpiWarps);
    }
    for (int d = 0; d < kSchedDepth; ++d) {
      mbar_init(&sfull_bar[d], 1);
      mbar_init(&sempty_bar[d], 1 + kEpiWarps);  // MMA lane + epilogue warps
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (PAIR == 2) tmem_alloc_pair<512>(tmem_holder);
    else tmem_alloc<512>(tmem_holder);
  }
  tc_fence_before();
  if constexpr (PAIR == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int units = args.m_tiles * args.n_tiles * args.splits;  // PAIR=2: m_tiles counts 256-row pair tiles
  const int ublk = PAIR == 2 ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int ugrid = PAIR == 2 ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
  // Tile scheduler.  Static: u = blockIdx.x + i*gridDim.x.  Dynamic (args.tile_counter):
  // the producer claims tiles with atomicAdd and hands them to the MMA / epilogue warps
  // through a small smem ring, so a kernel sharing the GPU with another stream's kernel
  // balances itself; the globally last claim resets the counter for the next launch.
  const bool dyn = args.tile_counter != nullptr;
  auto consumer_next = [&](uint32_t& slot, uint32_t& ph, int& u, bool first, bool is_mma) {
    if (!dyn) {
      u = first ? ublk : u + ugrid;
      return;
    }
    mbar_wait(&sfull_bar[slot], ph);
    u = *reinterpret_cast<volatile int32_t*>(&s_sched[slot]);
    if (is_mma) {
      mbar_arrive(&sempty_bar[slot]);
    } else {
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&sempty_bar[slot]);
    }
    if (++slot == kSchedDepth) { slot = 0; ph ^= 1; }
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, sslot = 0, sph = 0;
      for (int u = ublk;; u += ugrid) {
        if (dyn) {
          u = atomicAdd(args.tile_counter, 1);
          if (u == units + static_cast<int>(gridDim.x) - 1) atomicExch(args.tile_counter, 0);
          mbar_wait(&sempty_bar[sslot], sph ^ 1);
          s_sched[sslot] = u;
          mbar_arrive(&sfull_bar[sslot]);
          if (++sslot == kSchedDepth) { sslot = 0; sph ^= 1; }
        }
        if (u >= units) break;
        int mt, nt, sp;
        decode_unit(args, u, mt, nt, sp);
        const int kb0 = sp * args.kb_per_split;
        const int kb1 = min(args.kb_total, kb0 + args.kb_per_split);
        const int arow = (PAIR == 2 ? mt * 2 + static_cast<int>(rank) : mt) * BM;  // this CTA's A rows
        const int brow = nt * TBN + static_cast<int>(rank) * (TBN / PAIR);          // this CTA's B rows
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if constexpr (PAIR == 1) {
            mbar_arrive_expect_tx(&full_bar[stage], kStageBytes);
          } else if (rank == 0) {
            mbar_arrive_expect_tx(&full_bar[stage], 2 * kStageBytes);
          } else {
            mbar_arrive_cluster(mapa_shared(smem_u32(&full_bar[stage]), 0));
          }
          uint8_t* a = sA + stage * kSmemA;
          uint8_t* b = sB + stage * kSB;
          auto load = [&](const CUtensorMap* m, void* dst, int x, int y) {
            if constexpr (PAIR == 2) tma_load_2d_pair(m, &full_bar[stage], dst, x, y);
            else tma_load_2d(m, &full_bar[stage], dst, x, y);
          };
          if constexpr (!A_MN) {
            load(&tmA, a, kb * BK, arow);
          } else {
#pragma unroll
            for (int i = 0; i < BM / 64; ++i) load(&tmA, a + i * (BK * 128), arow + i * 64, kb * BK);
          }
          if constexpr (!B_MN) {
            load(&tmB, b, kb * BK, brow);
          } else {
#pragma unroll
            for (int i = 0; i < TBN / PAIR / 64; ++i) load(&tmB, b + i * (BK * 128), brow + i * 64, kb * BK);
          }
          if (++stage == kSt) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && rank == 0) {  // PAIR = 2: only the leader issues (cta_group::2)
      constexpr uint32_t idesc = umma_idesc_bf16(BM * PAIR, TBN, A_MN, B_MN);
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0, sslot = 0, sph = 0;
      int u = 0;
      for (bool first = true;; first = false) {
        consumer_next(sslot, sph, u, first, true);
        if (u >= units) break;
        int mt, nt, sp;
        decode_unit(args, u, mt, nt, sp);
        const int kb0 = sp * args.kb_per_split;
        const int kb1 = min(args.kb_total, kb0 + args.kb_per_split);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * kSmemA);
          const uint32_t b_base = smem_u32(sB + stage * kSB);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            if constexpr (PAIR == 2)
              umma_bf16_pair(d_tmem, operand_desc<A_MN>(a_base, k), operand_desc<B_MN>(b_base, k), idesc,
                             (kb > kb0 || k > 0) ? 1u : 0u);
            else
              umma_bf16(d_tmem, operand_desc<A_MN>(a_base, k), operand_desc<B_MN>(b_base, k), idesc,
                        (kb > kb0 || k > 0) ? 1u : 0u);
          }
          if constexpr (PAIR == 2) umma_commit_pair(&empty_bar[stage]);
          else umma_commit(&empty_bar[stage]);
          if (++stage == kSt) { stage = 0; phase ^= 1; }
        }
        if constexpr (PAIR == 2) umma_commit_pair(&tfull_bar[acc]);
        else umma_commit(&tfull_bar[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // 8 warps: warp w may only touch TMEM lanes 32*(w%4).. (its quadrant q); the two
    // warps of a quadrant split the tile's columns into [0, 128) and [128, TBN).
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int cbeg = half * (BN / 2);
    const int chalf_end = half ? TBN : BN / 2;
    uint32_t epi_chunk = 0;  // running count of bulk-store chunks (slot parity)
    uint32_t acc = 0, acc_phase = 0, sslot = 0, sph = 0;
    int u = 0;
    for (bool first = true;; first = false) {
      consumer_next(sslot, sph, u, first, false);
      if (u >= units) break;
      int mt, nt, sp;
      decode_unit(args, u, mt, nt, sp);
      if constexpr (PAIR == 2) mt = mt * 2 + static_cast<int>(rank);  // this CTA's 128-row half
      const int64_t row = static_cast<int64_t>(mt) * BM + q * 32 + lane;
      const bool row_ok = row < args.M;
      const int64_t col0 = static_cast<int64_t>(nt) * TBN;
      const int64_t rem = args.N - col0;
      const int ncols = rem < TBN ? static_cast<int>(rem) : TBN;
      const int cend = ncols < chalf_end ? ncols : chalf_end;  // this warp: [cbeg, cend)

      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);

      if constexpr (kFwd || kDz) {
        SupCursor cur;
        cur.idx = args.sup_idx + (row_ok ? row : 0) * args.k_max;
        cur.p = args.sup_p + (row_ok ? row : 0) * args.k_max;
        cur.k = row_ok ? args.k_max : 0;
        cur.limit = args.N;
        cur.gid0 = args.col_gid0;
        cur.seek(col0 + cbeg);
        float mrun = -INFINITY, srun = 0.f, usum = 0.f, rrun = 0.f;
        float coef = 0.f, lse2 = 0.f;
        if constexpr (kDz) {
          if (row_ok) {
            const float g = args.dloss ? __ldg(args.dloss) : 1.f;
            coef = g * __ldg(args.row_w + row);
            lse2 = __ldg(args.row_lse + row) * kLog2e;
          }
        }
        // F2 row mode: 0 Eq. 3 (support only), 1 reverse KL (+NTP through the support
        // {y: beta}), 2 dense KL(p_target || q) (empty support).
        int mode = 0;
        float lset2 = 0.f, eqzt = 0.f;
        const uint16_t* trow = nullptr;
        if constexpr (kT) {
          if (row_ok) {
            const uint8_t cls = __ldg(args.row_class + row);
            mode = (cls == AURORA_ROW_ACCEPT && args.f2_rkl) ? 1 : ((cls == AURORA_ROW_DISCARD && args.f2_dense) ? 2 : 0);
            trow = args.T + row * args.ldT;
            if (mode == 2) lset2 = __ldg(args.row_lse_t + row) * kLog2e;
            if (kDz && mode == 1) eqzt = __ldg(args.row_aux + row);
          }
        }
        if constexpr (kStage) {
          // A5 + the staged half of A7: pass 1 the exact max of this (row, tile half), pass 2
          // e = exp(z - m_half) -> s, the support dot u (and each support logit z_j, fp32,
          // for the backward's exact q_j - p~_j), and e rounded to bf16 into dZ^T[col][row]
          // (the backward rescales it in place by g w exp(m_half - lse) once lse is known).
          for (int cb = cbeg; cb < cend; cb += 32) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(taddr + cb, r);
            tmem_ld_wait();
            const int nj = (cb + 32 <= ncols) ? 32 : ncols - cb;
#pragma unroll
            for (int j = 0; j < 32; ++j) mrun = (j < nj) ? fmaxf(mrun, __uint_as_float(r[j])) : mrun;
          }
          const float mb = mrun * kLog2e;
          for (int cb = cbeg; cb < cend && mrun != -INFINITY; cb += 32) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(taddr + cb, r);
            tmem_ld_wait();
            const int nj = (cb + 32 <= ncols) ? 32 : ncols - cb;
            float z[32];
            float s0 = 0.f, s1 = 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) z[j] = __uint_as_float(r[j]);
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const float e0 = (j < nj) ? ex2_approx(fmaf(z[j], kLog2e, -mb)) : 0.f;
              const float e1 = (j + 1 < nj) ? ex2_approx(fmaf(z[j + 1], kLog2e, -mb)) : 0.f;
              s0 += e0;
              s1 += e1;
              if (row_ok) {
                __nv_bfloat16* dst = args.dzT + (col0 + cb + j) * args.ld_dzT + row;
                if (j < nj) dst[0] = __float2bfloat16_rn(e0);
                if (j + 1 < nj) dst[args.ld_dzT] = __float2bfloat16_rn(e1);
              }
            }
            srun += s0 + s1;
            while (cur.nxt < col0 + cb + 32) {
              const float zj = select32(z, static_cast<int>(cur.nxt - col0 - cb));
              usum = fmaf(cur.nxt_p, zj, usum);
              args.sup_z[row * args.k_max + cur.pos] = zj;
              cur.advance();
            }
          }
        } else
        for (int cb = cbeg; cb < cend; cb += 32) {  // warp-uniform bounds
          uint32_t r[32];
          tmem_ld_32x32b_x32(taddr + cb, r);
          const bool full = (cb + 32 <= ncols);
          float t[32];
          if constexpr (kT) {
            if (mode != 0) load_t32(trow, col0 + cb, full ? 32 : ncols - cb, args.t_vec, t);
          }
          tmem_ld_wait();
          float z[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) z[j] = __uint_as_float(r[j]);
          if constexpr (kFwd) {
            if (!full) {
#pragma unroll
              for (int j = 0; j < 32; ++j) z[j] = (cb + j < ncols) ? z[j] : -INFINITY;
            }
            float cmax = z[0];
#pragma unroll
            for (int j = 1; j < 32; ++j) cmax = fmaxf(cmax, z[j]);
            const float mnew = fmaxf(mrun, cmax);
            const float mb = mnew * kLog2e;
            const float scale = ex2_approx(mrun * kLog2e - mb);
            srun *= scale;
            float s0 = 0.f, s1 = 0.f;
            if (!kT || mode == 0) {
#pragma unroll
              for (int j = 0; j < 32; j += 2) {
                s0 += ex2_approx(fmaf(z[j], kLog2e, -mb));
                s1 += ex2_approx(fmaf(z[j + 1], kLog2e, -mb));
              }
            } else if (mode == 1) {  // r = sum e^{z-m} (z - t), rescaled with s
              rrun *= scale;
              float r0 = 0.f;
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const float e = ex2_approx(fmaf(z[j], kLog2e, -mb));
                s0 += e;
                r0 = fmaf(e, (cb + j < ncols) ? z[j] - t[j] : 0.f, r0);
              }
              rrun += r0;
            } else {  // u += sum_j p_j z_j, p_j = exp(t_j - lse_t)
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                s0 += ex2_approx(fmaf(z[j], kLog2e, -mb));
                if (cb + j < ncols) usum = fmaf(ex2_approx(fmaf(t[j], kLog2e, -lset2)), z[j], usum);
              }
            }
            srun += s0 + s1;
            mrun = mnew;
            while (cur.nxt < col0 + cb + 32) {
              usum = fmaf(cur.nxt_p, select32(z, static_cast<int>(cur.nxt - col0 - cb)), usum);
              cur.advance();
            }
          } else {
            if (!kT || mode == 0) {
#pragma unroll
              for (int j = 0; j < 32; ++j) z[j] = coef * ex2_approx(fmaf(z[j], kLog2e, -lse2));
            } else if (mode == 1) {  // q ((z - t) - E_q[z - t] + beta): RKL gradient + NTP's q
              const float base = args.ntp_beta - eqzt;
#pragma unroll
              for (int j = 0; j < 32; ++j) z[j] = coef * ex2_approx(fmaf(z[j], kLog2e, -lse2)) * (z[j] - t[j] + base);
            } else {  // q - p
#pragma unroll
              for (int j = 0; j < 32; ++j)
                z[j] = coef * (ex2_approx(fmaf(z[j], kLog2e, -lse2)) - ex2_approx(fmaf(t[j], kLog2e, -lset2)));
            }
            while (cur.nxt < col0 + cb + 32) {
              const int jj = static_cast<int>(cur.nxt - col0 - cb);
              const float sub = coef * cur.nxt_p;
#pragma unroll
              for (int j = 0; j < 32; ++j) z[j] = (j == jj) ? z[j] - sub : z[j];
              cur.advance();
            }
            if (row_ok) {
              __nv_bfloat16* dst = args.dzT + (col0 + cb) * args.ld_dzT + row;
              const int nj = full ? 32 : ncols - cb;
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (j < nj) dst[j * args.ld_dzT] = __float2bfloat16_rn(z[j]);
            }
          }
        }
        if constexpr (kFwd) {
          if (row_ok) {  // partial slot (vocab tile, column half); empty halves are neutral
            const int64_t o = row * (2 * args.n_tiles) + 2 * nt + half;
            args.p_max[o] = mrun;
            args.p_sum[o] = srun;
            args.p_u[o] = usum;
            if constexpr (kT) args.p_r[o] = rrun;
          }
        }
      } else if constexpr (EPI == EPI_SUMSQ) {
        // F3 pass 1: sum of squares of this warp's 32 rows x (up to) 128 columns, one partial
        // per (unit, CTA, epilogue warp) -- fixed slots and a fixed shuffle tree
        float acc2 = 0.f;
        for (int cb = cbeg; cb < cend; cb += 16) {
          uint32_t r[16];
          tmem_ld_32x32b_x16(taddr + cb, r);
          tmem_ld_wait();
          if (row_ok) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float x = (cb + j < ncols) ? __uint_as_float(r[j]) : 0.f;
              acc2 = fmaf(x, x, acc2);
            }
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc2 += __shfl_xor_sync(0xffffffffu, acc2, o);
        if (lane == 0) args.out[(static_cast<int64_t>(u) * PAIR + rank) * kEpiWarps + (warp - 2)] = acc2;
      } else if constexpr (EPI == EPI_STORE_BF16) {
        // bf16 output (F4 draft-layer projections): thread = row; each 32x32 block is packed
        // to bf16 (64 B per row) into a 64B-swizzled 2 KB slot and bulk-stored by TMA
        // (rows / columns outside the output are clipped by the tensor map).
        constexpr int kSlots = Plan::kSlots;
        uint8_t* slots = reinterpret_cast<uint8_t*>(stage_f32) + (warp - 2) * (kSlots * 2048);
        const int row0 = mt * BM + q * 32;
        for (int cb = cbeg; cb < cend; cb += 32) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(taddr + cb, r);
          uint8_t* slot = slots + (epi_chunk % kSlots) * 2048;
          if (lane == 0) bulk_wait_read<kSlots - 1>();
          __syncwarp();
          tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
            pk[j] = *reinterpret_cast<const uint32_t*>(&h2);
          }
          const uint32_t sbase = smem_u32(slot) + lane * 64;
          const uint32_t sw = (lane >> 1) & 3;
#pragma unroll
          for (int c = 0; c < 4; ++c)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sbase + ((c ^ sw) << 4)), "r"(pk[4 * c]),
                         "r"(pk[4 * c + 1]), "r"(pk[4 * c + 2]), "r"(pk[4 * c + 3])
                         : "memory");
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&tmC, slot, static_cast<int32_t>(col0 + cb), row0, 0);
            bulk_commit();
          }
          ++epi_chunk;
        }
      } else if (args.tma_store && !((args.dbg_epi & 4) && half == 1)) {  // EPI_STORE_F32, TMA bulk stores
        // thread = row; each 32x16 fp32 block goes to a 64B-swizzled smem slot (rows of
        // 64 B, 16 B chunk c of row r at chunk c ^ ((r >> 1) & 3): conflict-free 16 B
        // stores), then one lane issues a bulk tensor store (or reduce-add when
        // accumulating).  kSlots slots per warp in a ring; a slot is rewritten only after
        // the bulk engine has finished reading it (wait_group.read kSlots-1).
        constexpr int kSlots = Plan::kSlots > 0 ? Plan::kSlots : 1;
        uint8_t* slots = reinterpret_cast<uint8_t*>(stage_f32) + (warp - 2) * (kSlots * 2048);
        const int row0 = mt * BM + q * 32;
        const int dbg = args.dbg_epi;
        for (int cb = cbeg; cb < cend; cb += 16) {
          uint32_t r[16];
          if (!(dbg & 1)) tmem_ld_32x32b_x16(taddr + cb, r);
          else {
#pragma unroll
            for (int j = 0; j < 16; ++j) r[j] = static_cast<uint32_t>(cb + j);
          }
          uint8_t* slot = slots + (epi_chunk % kSlots) * 2048;
          if (lane == 0) bulk_wait_read<kSlots - 1>();
          __syncwarp();
          if (!(dbg & 1)) tmem_ld_wait();
          const uint32_t sbase = smem_u32(slot) + lane * 64;
          const uint32_t sw = (lane >> 1) & 3;
#pragma unroll
          for (int c = 0; c < 4; ++c)
            sts128(sbase + ((c ^ sw) << 4), __uint_as_float(r[4 * c]), __uint_as_float(r[4 * c + 1]),
                   __uint_as_float(r[4 * c + 2]), __uint_as_float(r[4 * c + 3]));
          if (dbg & 2) { __syncwarp(); ++epi_chunk; continue; }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int32_t x = static_cast<int32_t>(col0 + cb);
            if (args.accumulate) tma_reduce_add_3d(&tmC, slot, x, row0, sp);
            else if (dbg & 8) tma_store_3d_hint(&tmC, slot, x, row0, sp, l2_policy_evict_first());
            else tma_store_3d(&tmC, slot, x, row0, sp);
            bulk_commit();
          }
          ++epi_chunk;
        }
      } else {  // EPI_STORE_F32 through the LSU (fallback: unaligned output strides)
        // TMEM gives thread = row; transpose each 32x16 fp32 block through this warp's
        // smem slice so a store instruction writes eight full 64 B row segments.
        const uint32_t stg = smem_u32(reinterpret_cast<uint8_t*>(stage_f32) + (warp - 2) * (Plan::kSlots * 2048));
        float* obase = args.out + static_cast<int64_t>(sp) * args.split_stride;
        const bool vec_ok = ((args.ld_out & 3) == 0) && ((reinterpret_cast<uintptr_t>(obase) & 15) == 0);
        const int64_t row_base = static_cast<int64_t>(mt) * BM + q * 32;
        for (int cb = cbeg; cb < cend; cb += 16) {
          uint32_t r[16];
          tmem_ld_32x32b_x16(taddr + cb, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            sts128(stg + (lane * kStgLd + j) * 4, __uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                   __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
          __syncwarp();
#pragma unroll
          for (int it = 0; it < 4; ++it) {
            const int rl = it * 8 + (lane >> 2);
            const int cc = (lane & 3) * 4;
            const int64_t grow = row_base + rl;
            if (grow < args.M && cb + cc < ncols) {
              float4 v = lds128(stg + (rl * kStgLd + cc) * 4);
              float* dst = obase + grow * args.ld_out + col0 + cb + cc;
              if (vec_ok && cb + cc + 4 <= ncols) {
                if (args.accumulate) {
                  const float4 o = *reinterpret_cast<const float4*>(dst);
                  v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
                }
                *reinterpret_cast<float4*>(dst) = v;
              } else {
                const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  if (cb + cc + e < ncols) dst[e] = args.accumulate ? dst[e] + vv[e] : vv[e];
              }
            }
          }
          __syncwarp();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR == 2) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty_bar[acc]), 0));
        else mbar_arrive(&tempty_bar[acc]);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (((EPI == EPI_STORE_F32 && args.tma_store) || EPI == EPI_STORE_BF16) && lane == 0) bulk_wait<0>();
  }

  tc_fence_before();
  if constexpr (PAIR == 2) cluster_sync();
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (PAIR == 2) tmem_dealloc_pair<512>(tmem_base);
    else tmem_dealloc<512>(tmem_base);
  }
}

// ------------------------------------------------------------------ host side
namespace {
template <int EPI, bool A_MN, bool B_MN, int PAIR, int TBN = BN>
cudaError_t launch_impl(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC, const GemmArgs& args,
                        cudaStream_t s) {
  static bool attr_set = false;
  auto kern = k_umma_gemm<EPI, A_MN, B_MN, PAIR, TBN>;
  constexpr int kSmem = SmemPlan<EPI, A_MN, PAIR, TBN>::kBytes;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int units = args.m_tiles * args.n_tiles * args.splits;
  if (units <= 0) return cudaSuccess;
  static const int dbg_cluster = [] {
    const char* e = getenv("AURORA_DBG_CLUSTER1");
    return (e && e[0] == '1') ? 1 : 0;
  }();
  if (PAIR == 1 && dbg_cluster) {  // diagnostic: single-CTA tiles launched as 2-CTA clusters
    const int grid = units < kNumSMs ? ((units + 1) & ~1) : kNumSMs;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tmA, tmB, tmC, args);
    if (e != cudaSuccess) return e;
  } else if constexpr (PAIR == 1) {
    const int grid = units < kNumSMs ? units : kNumSMs;
    kern<<<grid, kGemmThreads, kSmem, s>>>(tmA, tmB, tmC, args);
  } else {
    const int pairs = units < kNumSMs / 2 ? units : kNumSMs / 2;
    static int max_clusters = -1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (max_clusters < 0) {
      cfg.gridDim = dim3(kNumSMs);
      if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess) max_clusters = 0;
      g_pair_max_clusters = max_clusters;
      cfg.gridDim = dim3(2 * pairs);
    }
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tmA, tmB, tmC, args);
    if (e != cudaSuccess) return e;
  }
  count_launch();
  return cudaGetLastError();
}
template <int PAIR>
cudaError_t dispatch(int epi, bool a_mn, bool b_mn, const CUtensorMap& tmA, const CUtensorMap& tmB,
                     const CUtensorMap& C, const GemmArgs& g, cudaStream_t s, int bn) {
  if constexpr (PAIR == 1) {
    if (bn != BN && (a_mn || b_mn || epi == EPI_STORE_F32)) return cudaErrorInvalidValue;
    if (bn == 224) {
      if (epi == EPI_FWD_STATS) return launch_impl<EPI_FWD_STATS, false, false, 1, 224>(tmA, tmB, C, g, s);
      if (epi == EPI_FWD_STAGE) return launch_impl<EPI_FWD_STAGE, false, false, 1, 224>(tmA, tmB, C, g, s);
      if (epi == EPI_BWD_DZ) return launch_impl<EPI_BWD_DZ, false, false, 1, 224>(tmA, tmB, C, g, s);
      if (epi == EPI_FWD_STATS_T) return launch_impl<EPI_FWD_STATS_T, false, false, 1, 224>(tmA, tmB, C, g, s);
      return launch_impl<EPI_BWD_DZ_T, false, false, 1, 224>(tmA, tmB, C, g, s);
    }
    if (bn == 192) {
      if (epi == EPI_FWD_STATS) return launch_impl<EPI_FWD_STATS, false, false, 1, 192>(tmA, tmB, C, g, s);
      if (epi == EPI_FWD_STAGE) return launch_impl<EPI_FWD_STAGE, false, false, 1, 192>(tmA, tmB, C, g, s);
      if (epi == EPI_BWD_DZ) return launch_impl<EPI_BWD_DZ, false, false, 1, 192>(tmA, tmB, C, g, s);
      if (epi == EPI_FWD_STATS_T) return launch_impl<EPI_FWD_STATS_T, false, false, 1, 192>(tmA, tmB, C, g, s);
      return launch_impl<EPI_BWD_DZ_T, false, false, 1, 192>(tmA, tmB, C, g, s);
    }
  }
  if (bn != BN) return cudaErrorInvalidValue;
  if (epi == EPI_FWD_STATS && !a_mn && !b_mn) return launch_impl<EPI_FWD_STATS, false, false, PAIR>(tmA, tmB, C, g, s);
  if (epi == EPI_FWD_STAGE && !a_mn && !b_mn) return launch_impl<EPI_FWD_STAGE, false, false, PAIR>(tmA, tmB, C, g, s);
  if (epi == EPI_BWD_DZ && !a_mn && !b_mn) return launch_impl<EPI_BWD_DZ, false, false, PAIR>(tmA, tmB, C, g, s);
  if (epi == EPI_FWD_STATS_T && !a_mn && !b_mn) return launch_impl<EPI_FWD_STATS_T, false, false, PAIR>(tmA, tmB, C, g, s);
  if (epi == EPI_SUMSQ && !a_mn && b_mn) return launch_impl<EPI_SUMSQ, false, true, PAIR>(tmA, tmB, C, g, s);
  if (epi == EPI_BWD_DZ_T && !a_mn && !b_mn) return launch_impl<EPI_BWD_DZ_T, false, false, PAIR>(tmA, tmB, C, g, s);
  if (epi == EPI_STORE_BF16) {
    if (!a_mn && !b_mn) return launch_impl<EPI_STORE_BF16, false, false, PAIR>(tmA, tmB, C, g, s);
    if (!a_mn && b_mn) return launch_impl<EPI_STORE_BF16, false, true, PAIR>(tmA, tmB, C, g, s);
    return cudaErrorInvalidValue;
  }
  if (epi == EPI_STORE_F32) {
    if (!a_mn && !b_mn) return launch_impl<EPI_STORE_F32, false, false, PAIR>(tmA, tmB, C, g, s);
    if (!a_mn && b_mn) return launch_impl<EPI_STORE_F32, false, true, PAIR>(tmA, tmB, C, g, s);
    if (a_mn && !b_mn) return launch_impl<EPI_STORE_F32, true, false, PAIR>(tmA, tmB, C, g, s);
    return launch_impl<EPI_STORE_F32, true, true, PAIR>(tmA, tmB, C, g, s);
  }
  return cudaErrorInvalidValue;
}
}  // namespace

cudaError_t launch_umma_gemm(int epi, bool a_mn, bool b_mn, const CUtensorMap& tmA, const CUtensorMap& tmB,
                             const GemmArgs& args, cudaStream_t s, const CUtensorMap* tmC, int pair, int bn) {
  static const CUtensorMap dummy{};
  const CUtensorMap& C = tmC ? *tmC : dummy;
  GemmArgs g = args;
  static const bool no_tma_store = [] {  // diagnostic: force the LSU store epilogue
    const char* e = getenv("AURORA_DBG_LSU_STORE");
    return e && e[0] == '1';
  }();
  g.tma_store = ((epi == EPI_STORE_F32 && !no_tma_store) || epi == EPI_STORE_BF16) && tmC ? 1 : 0;
  if (epi == EPI_STORE_BF16 && !tmC) return cudaErrorInvalidValue;
  static const int dbg_epi = [] {
    const char* e = getenv("AURORA_DBG_EPI");
    return e ? atoi(e) : 0;
  }();
  g.dbg_epi = dbg_epi;
  if (pair == 2) {
    g.tile_counter = nullptr;  // pairs use the static per-cluster schedule
    return dispatch<2>(epi, a_mn, b_mn, tmA, tmB, C, g, s, bn);
  }
  return dispatch<1>(epi, a_mn, b_mn, tmA, tmB, C, g, s, bn);
}

// ------------------------------------------------------------------ tensor maps
namespace {
using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}
}  // namespace

bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                    uint32_t box_inner, uint32_t box_outer) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 3D bf16 load map (SWIZZLE_128B) over [d2][d1][d0] (strides s1, s2 in elements), box
// {b0, b1, b2}; OOB elements are zero-filled.  Used by the tcgen05 tree-attention kernel.
bool make_tmap_bf16_3d(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                       uint64_t s2, uint32_t b0, uint32_t b1, uint32_t b2) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1 * 2, s2 * 2};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 3D bf16 output map [1][outer][inner], box {32, 32, 1}, SWIZZLE_64B (EPI_STORE_BF16).
bool make_tmap_bf16_out(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld * 2) % 16) return false;
  cuuint64_t dims[3] = {inner, outer, 1};
  cuuint64_t strides[2] = {ld * 2, ld * outer * 2};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_2d(CUtensorMap* map, int dtype, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                  uint32_t box_inner, uint32_t box_outer, int swizzle) {
  PFN_encodeTiled enc = get_encode();
  if (!enc || !base) return false;
  const uint64_t esz = dtype == 1 ? 4 : 2;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld * esz) % 16) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * esz};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = swizzle == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle == 64  ? CU_TENSOR_MAP_SWIZZLE_64B
                                : swizzle == 32  ? CU_TENSOR_MAP_SWIZZLE_32B
                                                 : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = enc(map, dtype == 1 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 3D fp32 output map [depth][outer][inner] (row stride ld floats, depth stride dstride
// floats), box {16, 32, 1}, SWIZZLE_64B.  Used by the TMA-store epilogue.
bool make_tmap_f32_out(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                       uint64_t depth, uint64_t dstride) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld * 4) % 16 || (dstride * 4) % 16) return false;
  cuuint64_t dims[3] = {inner, outer, depth};
  cuuint64_t strides[2] = {ld * 4, (depth > 1 ? dstride : ld * outer) * 4};
  cuuint32_t box[3] = {16, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace aur

// k_dw.cu — A8 (dW = dZ^T H) for small M: the A-resident CTA-pair sweep.
//
// At M = 384 the dW GEMM has K = M = 384: every 256x256 pair tile re-reads its operands
// (192 KB per CTA) from L2 to write 128 KB of fp32 output, and writes + operand re-reads
// share the L2's throughput.  Here a CTA pair owns one 256-row block of
// dZ^T (its unit): each CTA loads its 128 rows x K once into shared memory (K <= 512:
// <= 128 KB) and keeps them while it sweeps all d/256 column tiles, streaming only its
// half of H (128 columns x K) per tile.  Operand bytes per output byte drop from 1.5 to
// ~0.8.
//
// Warp roles as in k_umma_gemm (PAIR = 2): warp 0 TMA producer (A block once per unit,
// then the B ring), warp 1 the leader's single-thread tcgen05.mma.cta_group::2 issuer and
// TMEM owner, warps 2..9 the fp32 TMA-store epilogue (two 256-column accumulators).
// Barriers: a_full (A block landed in both CTAs, leader-side like the ring's full
// barriers), a_empty (all MMAs of the unit done: the A region may be reloaded; the
// commit is multicast to both CTAs).
#include "gemm_dev.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace aur {

namespace {
constexpr int kDwStages = 4;                       // B ring (16 KB per stage per CTA)
constexpr int kDwSB = (BN / 2) * BK * 2;           // B half per stage
constexpr int kDwMaxKb = 8;                        // K = M <= 512
constexpr int kDwARegion = kDwMaxKb * kSmemA;      // 128 KB
constexpr int kDwRing = kDwStages * kDwSB;         // 64 KB
constexpr int kDwStaging = kEpiWarps * 2 * 2048;   // 32 KB
constexpr int kDwSmem = kDwARegion + kDwRing + 1024 /*barriers*/ + 1024 /*align*/ + kDwStaging;
static_assert(kDwSmem <= 232448, "dynamic smem per CTA");
}  // namespace

__global__ void __launch_bounds__(kGemmThreads, 1)
    k_dw_resident(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const __grid_constant__ CUtensorMap tmC, const GemmArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                     // kb_total resident 128x64 K-major tiles
  uint8_t* sB = smem + kDwARegion;        // B ring
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sB + kDwRing);
  uint64_t* empty_bar = full_bar + kDwStages;
  uint64_t* tfull_bar = empty_bar + kDwStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* a_full = tempty_bar + 2;
  uint64_t* a_empty = a_full + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(a_empty + 1);
  float* stage_f32 = reinterpret_cast<float*>(sB + kDwRing + 1024);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int kb_total = args.kb_total;
  const int units = args.m_tiles;  // 256-row pair blocks of dZ^T
  const int n_tiles = args.n_tiles;
  const int ublk = static_cast<int>(blockIdx.x >> 1), ugrid = static_cast<int>(gridDim.x >> 1);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmC);
    for (int s = 0; s < kDwStages; ++s) {
      mbar_init(&full_bar[s], 2);  // leader: own expect_tx arrive + the peer's remote arrive
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 2 * kEpiWarps);
    }
    mbar_init(a_full, 2);
    mbar_init(a_empty, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_holder);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, a_phase = 0;
      for (int u = ublk; u < units; u += ugrid) {
        const int arow = (u * 2 + static_cast<int>(rank)) * BM;
        mbar_wait(a_empty, a_phase ^ 1);  // the previous unit's MMAs are done with A
        a_phase ^= 1;
        if (rank == 0) mbar_arrive_expect_tx(a_full, 2u * kb_total * kSmemA);
        else mbar_arrive_cluster(mapa_shared(smem_u32(a_full), 0));
        for (int kb = 0; kb < kb_total; ++kb) tma_load_2d_pair(&tmA, a_full, sA + kb * kSmemA, kb * BK, arow);
        for (int nt = 0; nt < n_tiles; ++nt) {
          const int bcol = nt * BN + static_cast<int>(rank) * (BN / 2);
          for (int kb = 0; kb < kb_total; ++kb) {
            mbar_wait(&empty_bar[stage], phase ^ 1);
            if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], 2u * kDwSB);
            else mbar_arrive_cluster(mapa_shared(smem_u32(&full_bar[stage]), 0));
            uint8_t* b = sB + stage * kDwSB;
#pragma unroll
            for (int i = 0; i < BN / 2 / 64; ++i)
              tma_load_2d_pair(&tmB, &full_bar[stage], b + i * (BK * 128), bcol + i * 64, kb * BK);
            if (++stage == kDwStages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader)
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM * 2, BN, false, true);
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0, a_phase = 0;
      for (int u = ublk; u < units; u += ugrid) {
        mbar_wait(a_full, a_phase);
        a_phase ^= 1;
        tc_fence_after();
        for (int nt = 0; nt < n_tiles; ++nt) {
          mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * BN;
          for (int kb = 0; kb < kb_total; ++kb) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            const uint32_t a_base = smem_u32(sA + kb * kSmemA);
            const uint32_t b_base = smem_u32(sB + stage * kDwSB);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_bf16_pair(d_tmem, operand_desc<false>(a_base, k), operand_desc<true>(b_base, k), idesc,
                             (kb > 0 || k > 0) ? 1u : 0u);
            umma_commit_pair(&empty_bar[stage]);
            if (++stage == kDwStages) { stage = 0; phase ^= 1; }
          }
          umma_commit_pair(&tfull_bar[acc]);
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1;
        }
        umma_commit_pair(a_empty);  // fires when every MMA of this unit has completed
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (TMA stores)
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int cbeg = half * (BN / 2);
    uint32_t epi_chunk = 0, acc = 0, acc_phase = 0;
    uint8_t* slots = reinterpret_cast<uint8_t*>(stage_f32) + (warp - 2) * (2 * 2048);
    for (int u = ublk; u < units; u += ugrid) {
      const int mt = u * 2 + static_cast<int>(rank);
      const int row0 = mt * BM + q * 32;
      for (int nt = 0; nt < n_tiles; ++nt) {
        const int64_t col0 = static_cast<int64_t>(nt) * BN;
        const int64_t rem = args.N - col0;
        const int ncols = rem < BN ? static_cast<int>(rem) : BN;
        const int cend = ncols < cbeg + BN / 2 ? ncols : cbeg + BN / 2;
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
        const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
        for (int cb = cbeg; cb < cend; cb += 16) {
          uint32_t r[16];
          tmem_ld_32x32b_x16(taddr + cb, r);
          uint8_t* slot = slots + (epi_chunk & 1) * 2048;
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
          tmem_ld_wait();
          const uint32_t sbase = smem_u32(slot) + lane * 64;
          const uint32_t sw = (lane >> 1) & 3;
#pragma unroll
          for (int c = 0; c < 4; ++c)
            sts128(sbase + ((c ^ sw) << 4), __uint_as_float(r[4 * c]), __uint_as_float(r[4 * c + 1]),
                   __uint_as_float(r[4 * c + 2]), __uint_as_float(r[4 * c + 3]));
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int32_t x = static_cast<int32_t>(col0 + cb);
            if (args.accumulate) tma_reduce_add_3d(&tmC, slot, x, row0, 0);
            else tma_store_3d(&tmC, slot, x, row0, 0);
            bulk_commit();
          }
          ++epi_chunk;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty_bar[acc]), 0));
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
    if (lane == 0) bulk_wait<0>();
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem_base);
  }
}

bool dw_resident_ok(int64_t kb_total) { return kb_total >= 1 && kb_total <= kDwMaxKb; }

cudaError_t launch_dw_resident(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                               const GemmArgs& args, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_dw_resident, cudaFuncAttributeMaxDynamicSharedMemorySize, kDwSmem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (args.m_tiles <= 0 || !dw_resident_ok(args.kb_total)) return cudaErrorInvalidValue;
  const int pairs = args.m_tiles < kNumSMs / 2 ? args.m_tiles : kNumSMs / 2;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = kDwSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_dw_resident, tmA, tmB, tmC, args);
  if (e != cudaSuccess) return e;
  count_launch();
  return cudaGetLastError();
}

}  // namespace aur

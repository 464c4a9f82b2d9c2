// k_dw_adamw.cu — NEXT F3 fused into A8: the lm_head's AdamW step applied straight from
// the dW GEMM's TMEM accumulators (P:487-489 global-norm clip 0.5, warm-up LR; P:495 fp32
// master weights and gradients).  dW = dZ^T H is recomputed on the tensor cores from the
// bf16 dZ^T the backward left in the workspace (K = M is small, so the MMAs are ~8% of
// the time) and never reaches HBM: per lm_head element the kernel moves m, v, W (fp32)
// in and out and the bf16 copy out — 26 B, the optimizer's compulsory traffic.
//
// One 2-CTA cluster per 256 x 256 dW tile (tcgen05.mma.cta_group::2), 11 warps per CTA:
//   warp 0      operand TMA (dZ^T K-major 128 x 64, H MN-major half 128 x 64), one stage (K = M
//               is 6-8 k-blocks per tile; the two TMEM accumulators hide the serial loads)
//   warp 1      TMEM allocation + the pair MMA issuer (leader CTA)
//   warps 2..9  epilogue: warp w owns TMEM lane quadrant w % 4 and half of the columns of
//               every state entry of that quadrant
//   warp 10     optimizer-state loader: TMA loads (SWIZZLE_128B) of m, v and the fp32 master W
//               into a 192 KB ring that runs ahead of the epilogue
// State entries (option dw_adamw_qe).  Default (1): 32 rows (one lane quadrant) x 128 columns,
// 48 KB, one ring slot per quadrant, consumed by that quadrant's two warps — every row segment
// a load or store touches is 512 B contiguous per array.  2: 32 x 64 (24 KB, two slots per
// quadrant).  0 (round-2 first version): 128 rows x 32 columns shared by all 8 warps (128 B row
// segments 4 d bytes apart: 5.24 TB/s of DRAM traffic, llama step 3.65 ms; quadrant entries:
// 3.51 ms).
// The epilogue updates each entry in place in shared memory (thread = row, conflict-free
// 16 B accesses through the swizzle), then reads it back transposed (full row segments per
// store instruction) and writes m, v, W (16 B) and the bf16 copy (8 B) with streaming stores,
// releasing the entry to the loader as soon as the values are in registers.  Measured and
// replaced: TMA bulk stores from the entry (every warp waited on cp.async.bulk.wait_group.read
// before the release: 5.06 TB/s), 16-column entries / a 3-entry ring (≈ 4.7 TB/s, latency-bound:
// bytes in flight per SM too few), spinning producer / MMA / loader waits (issue slots).
#include <cfloat>

#include "gemm_dev.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace aur {
namespace {

constexpr int kFWarps = 11;
constexpr int kFThreads = 32 * kFWarps;
constexpr int kFSt = 1;                               // operand stages (K = M: 6-8 k-blocks per tile;
                                                      // the TMEM double buffer hides the serial loads)
constexpr int kFSB = (BN / 2) * BK * 2;               // B half per CTA and stage
constexpr int kFStage = kSmemA + kFSB;                // 32 KB
constexpr int kECols = 32;                            // lm_head columns per state entry (128 B rows)
constexpr int kEArr = BM * kECols * 4;                // 16 KB: 128 rows x 32 fp32 (SW128)
constexpr int kEBytes = 3 * kEArr;                    // m, v, W
constexpr int kFR = 4;                                // state ring entries (3 in flight, 144 KB)
constexpr int kWCols = kECols / 2;                    // columns per epilogue warp and entry
constexpr int kEPerTile = BN / kECols;                // 8 entries per tile, each consumed by all 8 warps
// Quadrant entries (option dw_adamw_qe, QC = 128 or 64 columns): an entry is 32 rows (one TMEM
// lane quadrant) x QC columns (4 QC B contiguous per row and array: QC / 32 SW128 sub-blocks of
// 32 x 32 fp32), consumed by the two warps of that quadrant (QC / 2 columns each).  The ring
// holds the same 192 KB: QC = 128 gives every quadrant one 48 KB slot, QC = 64 two 24 KB slots.
constexpr int kQSub = 32 * 128;                       // 4 KB: 32 rows x 32 fp32 (SW128)
template <int QC>
struct QPlan {
  static constexpr int kArr = (QC / 32) * kQSub;      // bytes per array and entry
  static constexpr int kBytes = 3 * kArr;
  static constexpr int kSlots = (kFR * kEBytes) / kBytes;
  static constexpr int kPerTile = 4 * (BN / QC);      // entries per tile
  static constexpr int kWC = QC / 2;                  // columns per warp
  static constexpr int kCpr = kWC / 4;                // 16 B chunks per row and warp
  static_assert(kSlots % 4 == 0 && kSlots <= 8, "slots per quadrant");
};
constexpr int kRingOff = 0;
constexpr int kStateOff = kFSt * kFStage;
constexpr int kBarOff = kStateOff + kFR * kEBytes;
constexpr int kFSmem = kBarOff + 1024 + 1024;         // (16 entry barriers at most)         // barriers + base alignment
static_assert(kFSmem <= 232448, "dynamic smem per CTA");

struct Maps {
  CUtensorMap A, B;           // dZ^T (K-major, box 64 x 128), H (MN-major, box 64 x 64)
  CUtensorMap ml, vl, wl;     // fp32 [V, d] loads, box 32 x 128 (QE: 32 x 32), SW128
};

__device__ __forceinline__ void st_cs_v4(float* p, const float4& v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
// byte offset of (row r, 16 B chunk c) in a 128 B-row SWIZZLE_128B block
__device__ __forceinline__ uint32_t sw128(int r, int c) {
  return static_cast<uint32_t>(r * 128 + ((c ^ (r & 7)) << 4));
}

template <int QC>
__global__ void __launch_bounds__(kFThreads, 1)
    k_dw_adamw(const __grid_constant__ Maps mp, const DwAdamwArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem + kRingOff;
  uint8_t* sB = sA + kFSt * kSmemA;
  uint8_t* sState = smem + kStateOff;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kBarOff);
  uint64_t* empty_bar = full_bar + kFSt;
  uint64_t* tfull_bar = empty_bar + kFSt;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* efull_bar = tempty_bar + 2;   // state entries loaded
  uint64_t* eempty_bar = efull_bar + 8;  // state entries written back
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(eempty_bar + 8);
  constexpr bool QE = QC != 0;
  using QP = QPlan<QE ? QC : 128>;
  constexpr int kSlots = QE ? QP::kSlots : kFR;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mp.A);
    tma_prefetch_desc(&mp.B);
    tma_prefetch_desc(&mp.ml);
    tma_prefetch_desc(&mp.vl);
    tma_prefetch_desc(&mp.wl);
    for (int s = 0; s < kFSt; ++s) {
      mbar_init(&full_bar[s], 2);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 2 * kEpiWarps);
    }
    for (int e = 0; e < kSlots; ++e) {
      mbar_init(&efull_bar[e], 1);
      mbar_init(&eempty_bar[e], QE ? 2 : kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_holder);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  // static per-cluster schedule, n-fastest: the dZ^T rows of one vocab tile are read once
  const int units = args.m_tiles * args.n_tiles;
  const int ublk = static_cast<int>(blockIdx.x >> 1);
  const int ugrid = static_cast<int>(gridDim.x >> 1);
  auto decode = [&](int u, int& mt, int& nt) {
    nt = u % args.n_tiles;
    mt = u / args.n_tiles;
  };

  if (warp == 0) {
    // ---------------------------------------------------------------- operand TMA
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (int u = ublk; u < units; u += ugrid) {
        int mt, nt;
        decode(u, mt, nt);
        const int arow = (mt * 2 + static_cast<int>(rank)) * BM;
        const int brow = nt * BN + static_cast<int>(rank) * (BN / 2);
        for (int kb = 0; kb < args.kb_total; ++kb) {
          mbar_wait_sleep(&empty_bar[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], 2 * kFStage);
          else mbar_arrive_cluster(mapa_shared(smem_u32(&full_bar[stage]), 0));
          uint8_t* a = sA + stage * kSmemA;
          uint8_t* b = sB + stage * kFSB;
          tma_load_2d_pair(&mp.A, &full_bar[stage], a, kb * BK, arow);
#pragma unroll
          for (int i = 0; i < BN / 2 / 64; ++i)
            tma_load_2d_pair(&mp.B, &full_bar[stage], b + i * (BK * 128), brow + i * 64, kb * BK);
          if (++stage == kFSt) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- pair MMA issuer
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(2 * BM, BN, false, true);
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      for (int u = ublk; u < units; u += ugrid) {
        mbar_wait_sleep(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < args.kb_total; ++kb) {
          mbar_wait_sleep(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * kSmemA);
          const uint32_t b_base = smem_u32(sB + stage * kFSB);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16_pair(d_tmem, operand_desc<false>(a_base, k), operand_desc<true>(b_base, k), idesc,
                           (kb > 0 || k > 0) ? 1u : 0u);
          umma_commit_pair(&empty_bar[stage]);
          if (++stage == kFSt) { stage = 0; phase ^= 1; }
        }
        umma_commit_pair(&tfull_bar[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp == kFWarps - 1) {
    // ---------------------------------------------------------------- state loader
    if (lane == 0) {
      uint32_t pos = 0;
      for (int u = ublk; u < units; u += ugrid) {
        int mt, nt;
        decode(u, mt, nt);
        const int row0 = (mt * 2 + static_cast<int>(rank)) * BM;
        if constexpr (QE) {
          // entry order (column block cb, quadrant q): quadrant q's entries cycle through
          // slots q, q + 4, ...
          for (int cb = 0; cb < BN / QC; ++cb)
            for (int q = 0; q < 4; ++q, ++pos) {
              const uint32_t slot = pos % kSlots, ph = (pos / kSlots) & 1;
              mbar_wait_sleep(&eempty_bar[slot], ph ^ 1);
              mbar_arrive_expect_tx(&efull_bar[slot], QP::kBytes);
              uint8_t* dst = sState + slot * QP::kBytes;
              const int col = nt * BN + cb * QC, row = row0 + q * 32;
#pragma unroll
              for (int sb = 0; sb < QC / 32; ++sb) {
                tma_load_2d(&mp.ml, &efull_bar[slot], dst + sb * kQSub, col + sb * 32, row);
                tma_load_2d(&mp.vl, &efull_bar[slot], dst + QP::kArr + sb * kQSub, col + sb * 32, row);
                tma_load_2d(&mp.wl, &efull_bar[slot], dst + 2 * QP::kArr + sb * kQSub, col + sb * 32, row);
              }
            }
        } else {
          for (int e = 0; e < kEPerTile; ++e, ++pos) {
            const int col = nt * BN + e * kECols;
            const uint32_t slot = pos % kFR, ph = (pos / kFR) & 1;
            mbar_wait_sleep(&eempty_bar[slot], ph ^ 1);
            mbar_arrive_expect_tx(&efull_bar[slot], kEBytes);
            uint8_t* dst = sState + slot * kEBytes;
            tma_load_2d(&mp.ml, &efull_bar[slot], dst, col, row0);
            tma_load_2d(&mp.vl, &efull_bar[slot], dst + kEArr, col, row0);
            tma_load_2d(&mp.wl, &efull_bar[slot], dst + 2 * kEArr, col, row0);
          }
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int q = warp & 3;              // TMEM lane quadrant this warp may read
    const int half = (warp - 2) >> 2;    // 16-column half of every entry
    const float clip = __ldg(args.sc + 0), step_size = __ldg(args.sc + 1), isb2 = __ldg(args.sc + 2);
    const float decay = __ldg(args.sc + 3), b1 = __ldg(args.sc + 4), b2 = __ldg(args.sc + 5);
    const float eps = __ldg(args.sc + 6);
    const int r = q * 32 + lane;  // this thread's row within the CTA's 128-row block
    uint32_t acc = 0, acc_phase = 0, tile = 0;
    for (int u = ublk; u < units; u += ugrid, ++tile) {
      int mt, nt;
      decode(u, mt, nt);
      const int row0q = (mt * 2 + static_cast<int>(rank)) * BM + q * 32;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
      if constexpr (QE) {
        constexpr int kWC = QP::kWC, kCpr = QP::kCpr, kArr = QP::kArr;
        for (int cb = 0; cb < BN / QC; ++cb) {
          const int cl = cb * QC + half * kWC;  // tile-local column of this warp's kWC
          const uint32_t pos = tile * QP::kPerTile + cb * 4 + q;
          const uint32_t slot = pos % kSlots, ph = (pos / kSlots) & 1;
          uint32_t g[kWC / 32][32];
#pragma unroll
          for (int t = 0; t < kWC / 32; ++t) tmem_ld_32x32b_x32(taddr + cl + 32 * t, g[t]);
          mbar_wait(&efull_bar[slot], ph);
          tmem_ld_wait();
          const uint32_t base = smem_u32(sState + slot * QP::kBytes);
          const int sb0 = half * (kWC / 32);  // this warp's first sub-block
#pragma unroll
          for (int c = 0; c < kCpr; ++c) {
            const uint32_t o = (sb0 + (c >> 3)) * kQSub + sw128(lane, c & 7);
            float4 m4 = lds128(base + o), v4 = lds128(base + kArr + o), w4 = lds128(base + 2 * kArr + o);
            float* mm = &m4.x;
            float* vv = &v4.x;
            float* ww = &w4.x;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float gg = __uint_as_float(g[c >> 3][(4 * c + j) & 31]) * clip;
              mm[j] = fmaf(b1, mm[j], (1.f - b1) * gg);
              vv[j] = fmaf(b2, vv[j], (1.f - b2) * gg * gg);
              const float denom = sqrtf(vv[j]) * isb2 + eps;
              ww[j] = ww[j] * decay - step_size * (mm[j] / denom);
            }
            sts128(base + o, m4.x, m4.y, m4.z, m4.w);
            sts128(base + kArr + o, v4.x, v4.y, v4.z, v4.w);
            sts128(base + 2 * kArr + o, w4.x, w4.y, w4.z, w4.w);
          }
          __syncwarp();
          // transposed write-back: lane l -> (row (32 / kCpr) i + l / kCpr, 16 B chunk l % kCpr),
          // so each store instruction writes full 4 kWC B row segments
          const int64_t col = static_cast<int64_t>(nt) * BN + cl;
          const int cc = lane % kCpr;
#pragma unroll 4
          for (int i = 0; i < kCpr; ++i) {
            const int rr = i * (32 / kCpr) + lane / kCpr;
            const uint32_t o = (sb0 + (cc >> 3)) * kQSub + sw128(rr, cc & 7);
            const float4 m4 = lds128(base + o), v4 = lds128(base + kArr + o), w4 = lds128(base + 2 * kArr + o);
            const int64_t grow = row0q + rr;
            if (grow < args.V && col < args.d) {  // d % 64 == 0: a warp's columns are wholly in or out
              const int64_t gi = grow * args.d + col + cc * 4;
              st_cs_v4(args.m + gi, m4);
              st_cs_v4(args.v + gi, v4);
              st_cs_v4(args.w + gi, w4);
              const __nv_bfloat162 lo = __floats2bfloat162_rn(w4.x, w4.y), hi = __floats2bfloat162_rn(w4.z, w4.w);
              const uint32_t b0 = *reinterpret_cast<const uint32_t*>(&lo), b1 = *reinterpret_cast<const uint32_t*>(&hi);
              asm volatile("st.global.cs.v2.b32 [%0], {%1, %2};" ::"l"(args.wb + gi), "r"(b0), "r"(b1) : "memory");
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&eempty_bar[slot]);
        }
      } else
      for (int e = 0; e < kEPerTile; ++e) {
        const int cl = e * kECols + half * kWCols;  // tile-local column of this warp's 16
        const uint32_t pos = tile * kEPerTile + e;
        const uint32_t slot = pos % kFR, ph = (pos / kFR) & 1;
        uint32_t g[16];
        tmem_ld_32x32b_x16(taddr + cl, g);
        mbar_wait(&efull_bar[slot], ph);
        tmem_ld_wait();
        const uint32_t base = smem_u32(sState + slot * kEBytes);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t o = sw128(r, half * 4 + c);
          float4 m4 = lds128(base + o), v4 = lds128(base + kEArr + o), w4 = lds128(base + 2 * kEArr + o);
          float* mm = &m4.x;
          float* vv = &v4.x;
          float* ww = &w4.x;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float gg = __uint_as_float(g[4 * c + j]) * clip;
            mm[j] = fmaf(b1, mm[j], (1.f - b1) * gg);
            vv[j] = fmaf(b2, vv[j], (1.f - b2) * gg * gg);
            const float denom = sqrtf(vv[j]) * isb2 + eps;
            ww[j] = ww[j] * decay - step_size * (mm[j] / denom);
          }
          sts128(base + o, m4.x, m4.y, m4.z, m4.w);
          sts128(base + kEArr + o, v4.x, v4.y, v4.z, v4.w);
          sts128(base + 2 * kEArr + o, w4.x, w4.y, w4.z, w4.w);
        }
        __syncwarp();
        // transposed write-back with the LSU: lane l -> (row 8 i + l / 4, 16 B chunk l % 4), so
        // each store instruction writes eight full 64 B row segments; the entry is released
        // as soon as its values are in registers (no wait on a bulk-store read)
        const int64_t col = static_cast<int64_t>(nt) * BN + cl;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int rr = i * 8 + (lane >> 2), cc = lane & 3;
          const uint32_t o = sw128(q * 32 + rr, half * 4 + cc);
          const float4 m4 = lds128(base + o), v4 = lds128(base + kEArr + o), w4 = lds128(base + 2 * kEArr + o);
          const int64_t grow = row0q + rr;
          if (grow < args.V && col < args.d) {  // d % 64 == 0: an entry is wholly in or out
            const int64_t g = grow * args.d + col + cc * 4;
            st_cs_v4(args.m + g, m4);
            st_cs_v4(args.v + g, v4);
            st_cs_v4(args.w + g, w4);
            const __nv_bfloat162 lo = __floats2bfloat162_rn(w4.x, w4.y), hi = __floats2bfloat162_rn(w4.z, w4.w);
            const uint32_t b0 = *reinterpret_cast<const uint32_t*>(&lo), b1 = *reinterpret_cast<const uint32_t*>(&hi);
            asm volatile("st.global.cs.v2.b32 [%0], {%1, %2};" ::"l"(args.wb + g), "r"(b0), "r"(b1) : "memory");
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&eempty_bar[slot]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty_bar[acc]), 0));
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem_base);
  }
}

}  // namespace

bool dw_adamw_supported(int64_t V, int64_t d) { return V >= 1 && d % 64 == 0 && d >= 64; }

cudaError_t launch_dw_adamw(const void* dzT, int64_t ld_dzT, const void* H, int64_t M, int64_t d, int64_t V,
                            float* W_master, float* m, float* v, void* W_bf16, const float* sc, cudaStream_t s) {
  Maps mp;
  bool ok = make_tmap_bf16(&mp.A, dzT, M, V, ld_dzT, 64, BM) && make_tmap_bf16(&mp.B, H, d, M, d, 64, 64);
  const int qe = opt_dw_adamw_qe();  // 0: 128 x 32 entries; 1: 32 x 128; 2: 32 x 64
  const int box_rows = qe ? 32 : BM;
  ok = ok && make_tmap_2d(&mp.ml, 1, m, d, V, d, kECols, box_rows, 128) &&
       make_tmap_2d(&mp.vl, 1, v, d, V, d, kECols, box_rows, 128) &&
       make_tmap_2d(&mp.wl, 1, W_master, d, V, d, kECols, box_rows, 128);
  if (!ok) return cudaErrorInvalidValue;
  DwAdamwArgs a{};
  a.m_tiles = static_cast<int32_t>((V + 2 * BM - 1) / (2 * BM));
  a.n_tiles = static_cast<int32_t>((d + BN - 1) / BN);
  a.kb_total = static_cast<int32_t>((M + BK - 1) / BK);
  a.sc = sc;
  a.V = V;
  a.d = d;
  a.m = m;
  a.v = v;
  a.w = W_master;
  a.wb = static_cast<__nv_bfloat16*>(W_bf16);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_dw_adamw<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_dw_adamw<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_dw_adamw<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int units = a.m_tiles * a.n_tiles;
  const int pairs = units < kNumSMs / 2 ? units : kNumSMs / 2;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(kFThreads);
  cfg.dynamicSmemBytes = kFSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = qe == 1   ? cudaLaunchKernelEx(&cfg, k_dw_adamw<128>, mp, a)
                  : qe == 2 ? cudaLaunchKernelEx(&cfg, k_dw_adamw<64>, mp, a)
                            : cudaLaunchKernelEx(&cfg, k_dw_adamw<0>, mp, a);
  count_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace aur

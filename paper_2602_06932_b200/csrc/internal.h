// internal.h — host-side declarations shared by the library's translation units.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "../../include/aurora.h"

namespace aur {

constexpr int kNumSMs = 148;

// ---------------------------------------------------------------- GEMM engine
constexpr int BM = 128;  // tile rows (TMEM lanes)
constexpr int BN = 256;  // tile cols (TMEM columns per accumulator)
constexpr int BK = 64;   // K per pipeline stage (128 B of bf16 = one SW128 atom row)
constexpr int kStages = 4;
constexpr int kEpiWarps = 8;
constexpr int kGemmThreads = 64 + 32 * kEpiWarps;  // warp0 TMA, warp1 MMA, warps2-9 epilogue
constexpr int kSmemA = BM * BK * 2;
constexpr int kSmemB = BN * BK * 2;
constexpr int kSchedDepth = 4;  // tile-index ring depth (dynamic scheduler)
constexpr int kStgLd = 20;  // fp32 staging row stride (floats) for 32x16 blocks (LSU path)
constexpr int kGemmSmem = kStages * (kSmemA + kSmemB) + 1024 /*align*/ + 1024 /*barriers*/ + kEpiWarps * 2 * 2048;  // epilogue staging: 2 x (32x16 fp32) slots per warp

// *_T: the F2 objectives (reverse KL on ACCEPT rows, dense KL on DISCARD rows) — the
// epilogue also reads the row's target logits T (bf16) for the tile's columns.
// EPI_SUMSQ (F3 fused, norm pass): sum of squares of the output tile per (unit, CTA,
// epilogue warp); the output itself is never stored.
enum EpiKind : int {
  EPI_FWD_STATS = 0, EPI_BWD_DZ = 1, EPI_STORE_F32 = 2, EPI_FWD_STATS_T = 3, EPI_BWD_DZ_T = 4,
  EPI_SUMSQ = 5, EPI_FWD_STAGE = 6, EPI_STORE_BF16 = 7
};

// F3 hyperparameters (aurora_adamw_cfg_t as fp32 scalars).  The per-step scalars (warm-up
// LR, bias corrections, clip coefficient) are computed on the device by k_adamw_prep from
// the step (host value, or the device counter in the optimizer workspace) and the global
// norm, into a small float array `sc`: [0] clip, [1] step_size = lr_t / (1 - b1^t),
// [2] 1 / sqrt(1 - b2^t), [3] decay = 1 - lr_t wd, [4] b1, [5] b2, [6] eps.
struct AdamwHyper {
  float lr, beta1, beta2, eps, weight_decay, max_norm;
  int32_t warmup;
};
constexpr int kOptSc = 8;

// k_dw_adamw (F3 fused into the dW GEMM)
struct DwAdamwArgs {
  int32_t m_tiles, n_tiles, kb_total;
  const float* sc;
  int64_t V, d;
  float *m, *v, *w;    // fp32 [V, d] moments and master
  __nv_bfloat16* wb;   // bf16 [V, d] copy
};

struct GemmArgs {
  int32_t m_tiles, n_tiles, splits;
  int32_t kb_total, kb_per_split;
  int64_t M, N;  // valid extent of the GEMM output
  // ---- EPI_STORE_F32
  float* out;
  int64_t ld_out;
  int64_t split_stride;  // elements between split partial buffers
  int32_t accumulate;
  // ---- row-stat epilogues (fwd stats / bwd dz)
  const int32_t* sup_idx;  // [M, k_max] global ids, ascending, INT32_MAX padded
  const float* sup_p;
  int32_t k_max;
  int64_t col_gid0;  // global vocab id of GEMM column 0
  float* p_max;      // [M, 2*n_tiles] partial stats (fwd): one per (vocab tile, column half)
  float* p_sum;
  float* p_u;
  const float* row_lse;  // bwd
  const float* row_w;
  const float* dloss;    // nullable => 1
  __nv_bfloat16* dzT;    // [N_chunk, ld_dzT] transposed dLogits chunk (bwd)
  int64_t ld_dzT;
  int32_t* tile_counter;  // nullable: dynamic tile scheduler counter (zero before first use)
  int32_t n_fastest;      // tile raster: 0 = m-fastest (B streams once), 1 = n-fastest (A streams once)
  int32_t group;          // > 0: grouped raster, `group` m-tiles (group_on_n: n-tiles) per L2-resident group
  int32_t group_on_n;
  int32_t tma_store;      // set by launch_umma_gemm when an output tensor map is given
  int32_t dbg_epi;        // diagnostics only (AURORA_DBG_EPI): 1 skip tcgen05.ld, 2 skip fence + bulk store
  // ---- F2 objectives (EPI_*_T)
  const uint16_t* T;         // bf16 target logits of GEMM column 0, row stride ldT
  int64_t ldT;
  int32_t t_vec;             // T rows 16-byte aligned (vector loads)
  const uint8_t* row_class;
  int32_t f2_rkl;            // ACCEPT rows: reverse KL (+ NTP via the support {y: beta})
  int32_t f2_dense;          // DISCARD rows: dense KL(p_target || q)
  float ntp_beta;
  const float* row_lse_t;    // [M] log-sum-exp of the T row
  const float* row_aux;      // [M] E_q[z - t] (bwd, RKL rows)
  float* p_r;                // [M, 2*n_tiles] partial sum e^{z-m} (z - t) (fwd, RKL rows)
  float* sup_z;              // EPI_FWD_STAGE: [M, k_max] fp32 logit of each support entry hit
  // ---- F3 fused optimizer, norm pass (EPI_SUMSQ): one partial per (unit, CTA, warp) in `out`
};

// Launch the tcgen05 GEMM engine.  a_mn / b_mn select MN-major operands.
// tmC (optional, EPI_STORE_F32 only): fp32 output map from make_tmap_f32_out -> TMA-store
// epilogue (bulk stores / reduce-add); nullptr -> LSU store path.
// pair = 2: 2-CTA clusters with tcgen05.mma.cta_group::2 (M = 256 per pair tile; the
// caller sets args.m_tiles in 256-row units and builds K-major B maps with a 128-row box).
// bn: tile width, BN or (pair 1, K-major operands, EPI_FWD_STATS / EPI_BWD_DZ) 224 / 192;
// the caller sets args.n_tiles = cdiv(N, bn) and builds the B map with a bn-row box.
cudaError_t launch_umma_gemm(int epi, bool a_mn, bool b_mn, const CUtensorMap& tmA, const CUtensorMap& tmB,
                             const GemmArgs& args, cudaStream_t stream, const CUtensorMap* tmC = nullptr,
                             int pair = 1, int bn = BN);
bool make_tmap_f32_out(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                       uint64_t depth, uint64_t dstride);
// A8 for K = M <= 512 (k_dw.cu): CTA pairs keep their 128 rows of dZ^T resident and sweep
// every column tile.  args: m_tiles = 256-row pair blocks, n_tiles, kb_total, N, accumulate;
// tmA = dZ^T K-major (box 64x128), tmB = H MN-major (box 64x64), tmC = fp32 output map.
bool dw_resident_ok(int64_t kb_total);
cudaError_t launch_dw_resident(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                               const GemmArgs& args, cudaStream_t s);

// 2D bf16 tensor map (SWIZZLE_128B) over a row-major [outer, inner] matrix with row
// stride `ld` elements; box = {box_inner, box_outer}.
bool make_tmap_bf16_out(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld);
bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                    uint32_t box_inner, uint32_t box_outer);

bool make_tmap_bf16_3d(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                       uint64_t s2, uint32_t b0, uint32_t b1, uint32_t b2);

// ---------------------------------------------------------------- fused persistent bwd
enum BwdType : int { BT_DZ = 0, BT_DH = 1, BT_DW = 2 };
constexpr int kMaxChunks = 16;
struct BwdSeg {
  int32_t type, chunk, m_tiles, n_tiles, kb_total, kb_per_split, base, pad;
};
struct BwdMaps {
  CUtensorMap H_k, H_mn, W_k, W_mn, Z_k[2], Z_mn[2], O_W, O_H;
};
struct BwdArgs {
  int32_t nseg, total_units, nchunks;
  BwdSeg seg[3 * kMaxChunks];
  int64_t M, d, vocab_offset;
  int64_t c0[kMaxChunks], vc[kMaxChunks];
  int32_t n_dz[kMaxChunks], n_rd[kMaxChunks];
  const int32_t* sup_idx;
  const float* sup_p;
  int32_t k_max;
  const float* row_lse;
  const float* row_w;
  const float* dloss;
  __nv_bfloat16* dzT[2];
  int64_t ld_dzT;
  int32_t accumulate_dW;
  int32_t dh_m_tiles, dh_n_tiles;
  int32_t* tile_counter;
  int32_t* dz_done;
  int32_t* rd_done;
  int32_t* dh_flag;
};
cudaError_t launch_bwd_fused(const BwdMaps& maps, const BwdArgs& args, cudaStream_t s);

// ---------------------------------------------------------------- verify kernels
struct VerifyLaunch {
  const uint16_t* T;
  int64_t ldT, V_local, vocab_offset, V;
  int32_t M, R, N, k_max, nseg;
  int64_t seg_len;
  const int32_t* draft;
  const int32_t* parents;
  const int32_t* num_nodes;
  float* cand_val;      // [M, nseg, k_max]
  int32_t* cand_idx;
  float* top_val;       // [M, k_max] merged (value order); long path: [M, k_top]
  int32_t* top_idx;
  int32_t k_top;        // long-support path (k > AURORA_MAX_K): top-list length per row
  float* ept;           // F2: [M] E_p[t] of the target row (dense discard rows' H)
  float* lse_part;      // F2 x VP: [M, 3] this rank's (max, sum e^{t-m}, sum e^{t-m} t); null = final
  aurora_labels_t lab;
  aurora_loss_cfg_t cfg;
};
cudaError_t launch_target_scan(const VerifyLaunch& p, cudaStream_t s);
// persistent TMA-ring scan (16 B-aligned rows): writes scan_ring_lists() lists per (row, segment)
bool scan_ring_ok(const VerifyLaunch& p);
int scan_ring_lists();
cudaError_t launch_target_scan_ring(const VerifyLaunch& p, cudaStream_t s);
// load-balanced flat scan (scan_flat_ok): equal contiguous vector ranges per warp, `*nlists`
// (= scan_flat_slots) lists per row in cand_val / cand_idx
constexpr int kScanFlatCtas = 2;
bool scan_flat_ok(const VerifyLaunch& p);
int scan_flat_slots(int64_t M, int64_t V_local);
cudaError_t launch_target_scan_flat(const VerifyLaunch& p, int* nlists, cudaStream_t s);
cudaError_t launch_topk_merge(const VerifyLaunch& p, const float* in_val, const int32_t* in_idx, int nlists,
                              int64_t row_stride, int64_t list_stride, cudaStream_t s);
cudaError_t launch_target_scan_topk(const VerifyLaunch& p, const int32_t* tk_idx, const uint16_t* tk_val, int32_t K_t,
                                    cudaStream_t s);
cudaError_t launch_verify(const VerifyLaunch& p, cudaStream_t s);
cudaError_t launch_finalize(const VerifyLaunch& p, cudaStream_t s);
// Long supports (F1 soft distillation, k up to AURORA_MAX_K_SPARSE): CTA per row.
cudaError_t launch_sort_pairs(const VerifyLaunch& p, const int32_t* tk_idx, const uint16_t* tk_val, int32_t K_t,
                              cudaStream_t s);
cudaError_t launch_finalize_long(const VerifyLaunch& p, cudaStream_t s);
// F2: per-row log-sum-exp and E_p[t] of the dense target row (CTA per row).
cudaError_t launch_row_lse_t(const VerifyLaunch& p, cudaStream_t s);
cudaError_t launch_row_lse_t_combine(const VerifyLaunch& p, const float* parts /*[P,M,3]*/, int P, cudaStream_t s);

// ---------------------------------------------------------------- row kernels
// msu rows are (m, s, u, r): r = sum e^{z-m} (z - t) on F2 RKL rows (pr nullable => 0).
constexpr int kMsu = 4;
cudaError_t launch_reduce_partials(const float* pm, const float* ps, const float* pu, const float* pr, int64_t M,
                                   int n_tiles, float* msu /*[M,kMsu]*/, cudaStream_t s);
struct RowF2 {  // F2 objectives in the row combine (all zero / null: Eq. 3 FKL everywhere)
  int32_t rkl;
  float beta;
  const float* row_lse_t;
  float* row_aux;  // out: E_q[z - t] on RKL rows; the support log-sum-exp on restricted rows
  int32_t restricted;        // DISCARD rows: SPEC's restricted softmax over the support
  const float* sup_z;        // [M, k_max] support logits (staged forward)
  const int32_t* sup_idx;    // [M, k_max] (INT32_MAX = padding)
  int32_t k_max;
};
cudaError_t launch_row_combine(const float* msu_all /*[P,M,kMsu]*/, int P, int64_t M, const float* row_H,
                               const float* row_w, const uint8_t* row_class, float* row_lse, float* row_loss,
                               float* block_partials, int* nblocks_out, const RowF2& f2, cudaStream_t s);
cudaError_t launch_loss_sum(const float* block_partials, int nblocks, float* loss, cudaStream_t s);
cudaError_t launch_splitk_reduce(const float* partials, int splits, int64_t n_elems, float* out, int accumulate,
                                 cudaStream_t s);
cudaError_t launch_dz_rescale(__nv_bfloat16* dzT, int64_t ld, int64_t M, int64_t V_local, int bn, int n_tiles,
                              const float* pm, const float* row_lse, const float* row_w, const float* dloss,
                              const uint8_t* row_class, int restricted, cudaStream_t s);
cudaError_t launch_dz_support_fix(__nv_bfloat16* dzT, int64_t ld, int64_t M, int64_t V_local, int64_t vocab_offset,
                                  const aurora_labels_t* lab, const float* sup_z, const float* row_lse,
                                  const float* dloss, int restricted, cudaStream_t s);
cudaError_t launch_debug_dlogits(const __nv_bfloat16* H, const __nv_bfloat16* W, int64_t M, int64_t d,
                                 int64_t V_local, int64_t vocab_offset, const aurora_labels_t* lab,
                                 const float* row_lse, const float* dloss, const int32_t* rows, int n_rows,
                                 float* out, cudaStream_t s);

// ---------------------------------------------------------------- F3 optimizer
int adamw_partials();
// ordered sum of n partials (+ extra_sq) -> out[0] (one CTA)
cudaError_t launch_sum_partials(const float* partials, int nparts, float* out, cudaStream_t s);
cudaError_t launch_sumsq(const float* g, int64_t n, float* partials, float* norm_sq, cudaStream_t s);
cudaError_t launch_dot(const float* a, const float* b, int64_t n, float* partials, float* out, cudaStream_t s);
// per-step scalars (see AdamwHyper): host_step >= 1, or 0 = increment and use *step_dev
cudaError_t launch_adamw_prep(const float* norm_sq, const float* extra_sq, const AdamwHyper& h, int64_t host_step,
                              int64_t* step_dev, float* sc, float* grad_norm, cudaStream_t s);
cudaError_t launch_adamw(float* W, void* Wb, float* m, float* v, const float* g, int64_t n, const float* sc,
                         cudaStream_t s);
bool dw_adamw_supported(int64_t V, int64_t d);
cudaError_t launch_dw_adamw(const void* dzT, int64_t ld_dzT, const void* H, int64_t M, int64_t d, int64_t V,
                            float* W_master, float* m, float* v, void* W_bf16, const float* sc, cudaStream_t s);
// generic 2-D map: dtype 0 bf16 / 1 fp32, dims {inner, outer}, row stride ld elements,
// box {box_inner, box_outer}, swizzle 0 / 32 / 64 / 128 bytes
bool make_tmap_2d(CUtensorMap* map, int dtype, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                  uint32_t box_inner, uint32_t box_outer, int swizzle);

// ---------------------------------------------------------------- accounting
extern std::atomic<uint64_t> g_launches;
extern int g_pair_max_clusters;  // cudaOccupancyMaxActiveClusters of the CTA-pair GEMM (-1: unknown)
inline void count_launch(int n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Phase profiling (CUDA events on the caller's stream).
enum Phase : int { PH_SCAN = 0, PH_VERIFY, PH_FWD_GEMM, PH_FWD_COMBINE, PH_BWD_DZ, PH_BWD_DW, PH_BWD_DH,
                   PH_BWD_REDUCE, PH_COMM, PH_BWD_FUSED, PH_OPTIM, PH_TREE_FWD, PH_TREE_BWD_DQ,
                   PH_TREE_BWD_DKDV, PH_TREE_BWD_FUSED, PH_TREE_FWD_TC, PH_BWD_RESCALE, PH_COUNT };
void prof_begin(int phase, cudaStream_t s);
int opt_tree_bwd_split();  // aurora_set_option("tree_bwd_split")
int opt_tree_fwd_tc();     // aurora_set_option("tree_fwd_tc")
int opt_tree_bwd_tc();     // aurora_set_option("tree_bwd_tc")
int opt_dw_adamw_qe();     // aurora_set_option("dw_adamw_qe")
void prof_end(int phase, cudaStream_t s);

}  // namespace aur

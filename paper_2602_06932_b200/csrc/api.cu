// api.cu — the extern "C" boundary (include/aurora.h): validation, workspace carving,
// tensor maps, kernel sequencing and the NCCL collectives of the VP/DP modes.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "comm.h"
#include "internal.h"

namespace aur {

std::atomic<uint64_t> g_launches{0};

// ------------------------------------------------------------------ profiling
namespace {
std::mutex g_prof_mu;
bool g_prof_on = false;
struct ProfRec { int phase; cudaEvent_t a, b; };
std::vector<ProfRec> g_prof_open, g_prof_done;
std::vector<cudaEvent_t> g_ev_pool;
cudaEvent_t ev_get() {
  if (!g_ev_pool.empty()) { cudaEvent_t e = g_ev_pool.back(); g_ev_pool.pop_back(); return e; }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
const char* kPhaseNames[PH_COUNT] = {"target_scan", "verify", "fwd_gemm", "fwd_combine", "bwd_dz_gemm",
                                     "bwd_dw_gemm", "bwd_dh_gemm", "bwd_reduce", "comm", "bwd_fused", "adamw",
                                     "tree_attn_fwd", "tree_attn_bwd_dq", "tree_attn_bwd_dkdv",
                                     "tree_attn_bwd_fused", "tree_attn_fwd_tc", "bwd_dz_rescale"};
}  // namespace

// Inside a CUDA-graph capture the phase events become external event-record nodes, so
// every replay re-records them and they stay readable (aurora_profile_peek).
void prof_record(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
  else
    cudaEventRecord(e, s);
}
void prof_begin(int phase, cudaStream_t s) {
  if (!g_prof_on) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  ProfRec r{phase, ev_get(), ev_get()};
  prof_record(r.a, s);
  g_prof_open.push_back(r);
}
void prof_end(int phase, cudaStream_t s) {
  if (!g_prof_on) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (size_t i = g_prof_open.size(); i-- > 0;) {
    if (g_prof_open[i].phase == phase) {
      prof_record(g_prof_open[i].b, s);
      g_prof_done.push_back(g_prof_open[i]);
      g_prof_open.erase(g_prof_open.begin() + static_cast<long>(i));
      return;
    }
  }
}

}  // namespace aur

namespace aur {
namespace {

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t rup(int64_t a, int64_t b) { return cdiv(a, b) * b; }
inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

aurora_status_t cuda_status(cudaError_t e) { return e == cudaSuccess ? AURORA_OK : AURORA_ERR_CUDA; }

// ---- workspace layout: one carve routine used by both sizing and the calls
struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base(static_cast<char*>(b)) {}
  template <typename T>
  T* take(int64_t n) {
    off = rup(static_cast<int64_t>(off), 256);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += static_cast<size_t>(n) * sizeof(T);
    return p;
  }
};

// ---- tuning options (aurora_set_option); defaults from the environment
struct Options {
  int gemm_pair = 0;       // 0 auto, 1 single-CTA tiles, 2 CTA-pair tiles
  int bwd_mode = 0;        // 0 classic per-chunk launches, 1 fused persistent kernel
  int bwd_concurrent = 0;  // classic mode: dW || dH on side streams (measured equal to serial; off
                           // by default so per-kernel event timings stay clean)
  int tile_n = 0;          // fwd / dz tile width: 0 auto, else 256 / 224 / 192
  int64_t dz_chunk_bytes = int64_t(16) << 30;  // classic bwd: dZ^T chunk budget (bytes; 16 GiB of the
                                                // 180 GB HBM: the tree config's 7.8 GB in one chunk)
  int scan_ctas = 2;                           // target-scan CTAs per SM (segments per row)
  int tree_fwd_tc = 2;                         // F4 fwd when G*(N+1) <= 128: 2 (default) = one-pass tcgen05
                                               // kernel, two work items per SM; 3 = one item, deep rings;
                                               // 1 = two-pass tcgen05; 0 = mma.sync
  int tree_bwd_tc = 1;                         // F4 bwd when G*(N+1) <= 128: 1 (default) = tcgen05 kernel,
                                               // 0 = mma.sync fused kernel
  int tree_bwd_split = 0;                      // F4 bwd: 1 = separate dQ / dK-dV kernels even when the
                                               // fused one applies (A/B and coverage of the general path)
  int dw_resident = 0;                         // dW with K = M <= 512: A-resident pair sweep (measured
                                               // slower at M = 384: 0.507 vs 0.470 ms; opt-in)
  int gram_norm = 1;                           // F3 fused: Gram-form global norm when M is small
  int dw_adamw_qe = 1;                         // F3 fused state entries: 0 = 128 x 32, 1 = 32 x 128, 2 = 32 x 64
  int debug_gemm_group = 0;                    // aurora_debug_gemm only: grouped raster (< 0: groups of n-tiles)
  int scan_flat = 1;                           // A2: 1 = load-balanced flat scan (equal vector ranges per warp)
  int scan_ring = 0;                           // A2: 1 = persistent TMA-ring scan (measured slower: opt-in)
  int fwd_stage = 1;                           // Eq. 3: the fwd stages exp(z - m_half) in dZ^T so the
                                               // bwd needs no recompute GEMM (0: recompute, round-1 path)
  Options() {
    if (const char* e = getenv("AURORA_FWD_STAGE")) fwd_stage = atoi(e) ? 1 : 0;
    if (const char* e = getenv("AURORA_SCAN_RING")) scan_ring = atoi(e) ? 1 : 0;
    if (const char* e = getenv("AURORA_SCAN_FLAT")) scan_flat = std::min(2, std::max(0, atoi(e)));
    if (const char* e = getenv("AURORA_DW_ADAMW_QE")) dw_adamw_qe = std::min(2, std::max(0, atoi(e)));
    if (const char* e = getenv("AURORA_DW_RESIDENT")) dw_resident = atoi(e) ? 1 : 0;
    if (const char* e = getenv("AURORA_SCAN_CTAS")) scan_ctas = std::max(1, atoi(e));
    if (const char* e = getenv("AURORA_DZ_CHUNK_BYTES")) dz_chunk_bytes = atoll(e);
    if (const char* e = getenv("AURORA_TILE_N")) tile_n = atoi(e);
    if (const char* e = getenv("AURORA_PAIR")) gemm_pair = atoi(e);
    if (const char* e = getenv("AURORA_BWD")) bwd_mode = std::strcmp(e, "fused") == 0 ? 1 : 0;
    if (const char* e = getenv("AURORA_SERIAL_BWD")) bwd_concurrent = (e[0] == '0') ? 1 : 0;
    if (const char* e = getenv("AURORA_TREE_FWD_TC")) tree_fwd_tc = std::min(3, std::max(0, atoi(e)));
    if (const char* e = getenv("AURORA_TREE_BWD_SPLIT")) tree_bwd_split = atoi(e) ? 1 : 0;
    if (const char* e = getenv("AURORA_TREE_BWD_TC")) tree_bwd_tc = atoi(e) ? 1 : 0;
  }
};
Options& opts() {
  static Options o;
  return o;
}
// CTA-pair tiles (256 rows) when the GEMM's row count pads to 256 with little waste.
int pair_for(int64_t rows) {
  if (opts().gemm_pair == 1) return 1;
  if (opts().gemm_pair == 2) return 2;
  return (rows % 256 == 0 || rows >= 4096) ? 2 : 1;
}
// Tile width for the K-major fwd / dz GEMMs (single-CTA tiles only).  A persistent CTA
// does ceil(tiles / 148) tiles, each costing ~(width + a fixed per-tile overhead, measured
// ~160 columns' worth: operand refill of A, epilogue tail): pick the width with the least
// per-SM cost, 256 unless a narrower one is >= 2% better.  (M = 384, one 32K-column chunk:
// 224 wins, 2.55 -> 2.92 waves; the whole 128K vocabulary at once: 256 wins.)
constexpr int kTileWidths[3] = {256, 224, 192};
constexpr int kMinBN = 192;
constexpr int kTileOverheadCols = 160;
int kmajor_bn(int64_t m_tiles, int64_t N, int pair) {
  if (pair != 1) return BN;
  if (opts().tile_n) return opts().tile_n;
  auto cost = [&](int bn) {
    return static_cast<double>(cdiv(m_tiles * cdiv(N, bn), kNumSMs)) * (bn + kTileOverheadCols);
  };
  int best = BN;
  double best_cost = cost(BN);
  for (int bn : kTileWidths) {
    const double c = cost(bn);
    if (c < 0.98 * best_cost) { best = bn; best_cost = c; }
  }
  return best;
}
// Scan segments per row: enough (row, segment) CTAs for `scan_ctas` per SM; long segments
// amortise the per-CTA warm start and list merge (measured: 32K-column segments spent most
// of their instructions there).
int scan_nseg(int64_t M, int64_t V_local) {
  int64_t nseg = cdiv(static_cast<int64_t>(opts().scan_ctas) * kNumSMs, std::max<int64_t>(M, 1));
  nseg = std::min<int64_t>(nseg, 32);
  nseg = std::min<int64_t>(nseg, cdiv(V_local, 2048));
  return static_cast<int>(std::max<int64_t>(nseg, 1));
}
// dLogits chunk width.  The bf16 dZ^T of the whole local vocabulary is M x V_local x 2 B
// (Llama: 98 MB of the 180 GB HBM): keep it whole when it fits the chunk budget (option
// "dz_chunk_bytes", default 16 GiB) so the bwd is one dz, one dW and one dH launch with no
// per-chunk wave tails; otherwise the fewest equal chunks that fit (<= 20), rounded to 256.
int64_t chunk_cols(int64_t V_local, int64_t M) {
  const int64_t per_col = rup(M, 8) * 2;
  int64_t n = cdiv(V_local * per_col, std::max<int64_t>(opts().dz_chunk_bytes, per_col * 256));
  n = std::min<int64_t>(std::max<int64_t>(n, 1), 20);
  return std::min(rup(cdiv(V_local, n), 256), rup(V_local, 256));
}
// split-K factor for dH: the (m, n) tile count is small (M x d output) so pick the
// split that fills whole waves of 148 SMs best (fewest splits within 3% of the best).
int dh_splits(int64_t M, int64_t d, int64_t kb_total, int pair = 1) {
  const int64_t tiles = cdiv(M, BM * pair) * cdiv(d, BN);
  const int64_t slots = kNumSMs / pair;
  double best_eff = 0.0;
  double eff[17] = {0};
  for (int64_t s = 1; s <= 8 && s <= kb_total; ++s) {
    const int64_t units = tiles * s;
    eff[s] = static_cast<double>(units) / static_cast<double>(cdiv(units, slots) * slots);
    best_eff = std::max(best_eff, eff[s]);
  }
  for (int64_t s = 1; s <= 8 && s <= kb_total; ++s)
    if (eff[s] >= best_eff - 0.03) return static_cast<int>(cdiv(kb_total, cdiv(kb_total, s)));
  return 1;
}

struct VerifyWs { float* cand_val; int32_t* cand_idx; float* top_val; int32_t* top_idx; float* ept; float* lse_part; };
// TMA-ring scan: one warp per (row, segment) item; enough items for 2 per warp slot of the grid
// (148 x 8 warps), segments >= 16K columns (one top-k list per segment), <= 32 per row
int ring_nseg(int64_t M, int64_t V_local) {
  int64_t nseg = cdiv(2 * kNumSMs * 8, std::max<int64_t>(M, 1));
  nseg = std::min<int64_t>(nseg, std::max<int64_t>(1, V_local / 16384));
  return static_cast<int>(std::min<int64_t>(std::max<int64_t>(nseg, 1), 32));
}
VerifyWs carve_verify(Carver& c, int64_t M, int64_t V_local, int k_max) {
  const int nseg = std::max({scan_nseg(M, V_local), ring_nseg(M, V_local) * scan_ring_lists(),
                             scan_flat_slots(M, V_local)});
  VerifyWs w;
  w.ept = c.take<float>(M);
  w.lse_part = c.take<float>(M * 3);
  w.cand_val = c.take<float>(M * nseg * k_max);
  w.cand_idx = c.take<int32_t>(M * nseg * k_max);
  w.top_val = c.take<float>(M * k_max);
  w.top_idx = c.take<int32_t>(M * k_max);
  return w;
}
VerifyWs carve_verify_long(Carver& c, int64_t M, int k_top) {  // F1 long supports: top lists only
  VerifyWs w{};
  w.top_val = c.take<float>(M * k_top);
  w.top_idx = c.take<int32_t>(M * k_top);
  return w;
}
struct FwdWs { float *pm, *ps, *pu, *pr, *msu, *bp; };
FwdWs carve_fwd(Carver& c, int64_t M, int64_t V_local) {
  FwdWs w;
  const int64_t max_tiles = cdiv(V_local, kMinBN);  // sized for the narrowest tile width
  w.pm = c.take<float>(M * 2 * max_tiles);  // one partial per (vocab tile, column half)
  w.ps = c.take<float>(M * 2 * max_tiles);
  w.pu = c.take<float>(M * 2 * max_tiles);
  w.pr = c.take<float>(M * 2 * max_tiles);  // F2 reverse-KL partials
  w.msu = c.take<float>(M * kMsu);
  w.bp = c.take<float>(cdiv(M, 256) + 1);
  return w;
}
constexpr int kCounters = 64;  // dynamic-scheduler tile counters (one per launch in a call)
struct BwdWs { int32_t* counters; __nv_bfloat16* dzT; float* dh_part; int64_t vc, m_pad; int splits; };
BwdWs carve_bwd(Carver& c, int64_t M, int64_t d, int64_t V_local) {
  BwdWs w;
  w.counters = c.take<int32_t>(kCounters);
  w.vc = chunk_cols(V_local, M);
  w.m_pad = rup(M, 8);
  w.dzT = c.take<__nv_bfloat16>(w.vc * w.m_pad);
  w.splits = dh_splits(M, d, cdiv(w.vc, BK), pair_for(M));
  w.dh_part = w.splits > 1 ? c.take<float>(static_cast<int64_t>(w.splits) * M * d) : nullptr;
  return w;
}

// ---- fused bwd layout: counters, two 1/8-vocab dZ^T buffers, dH split partials
int64_t fused_chunk_cols(int64_t V_local) {
  if (V_local <= 8 * BN) return rup(cdiv(V_local, 2), BN);
  return rup(cdiv(V_local, 8), BN);
}
int fused_dh_splits(int64_t M, int64_t d, int64_t kb_total) {
  const int64_t tiles = cdiv(M, BM) * cdiv(d, BN);
  int64_t s = std::min<int64_t>(std::max<int64_t>(cdiv(kNumSMs, tiles), 1), 8);
  return static_cast<int>(std::max<int64_t>(std::min<int64_t>(s, kb_total), 1));
}
struct FusedWs {
  int32_t* counters;  // [0] tile counter, [1..16] dz_done, [17..32] rd_done, [33..] dh flags
  int n_counters;
  __nv_bfloat16* dzT[2];
  float* dh_part;
  int64_t vc, m_pad;
  int splits;
};
FusedWs carve_fused(Carver& c, int64_t M, int64_t d, int64_t V_local) {
  FusedWs w;
  w.vc = fused_chunk_cols(V_local);
  w.m_pad = rup(M, 8);
  w.splits = fused_dh_splits(M, d, cdiv(w.vc, BK));
  w.n_counters = 1 + 2 * kMaxChunks + static_cast<int>(cdiv(M, BM) * cdiv(d, BN)) * w.splits;
  w.counters = c.take<int32_t>(w.n_counters);
  w.dzT[0] = c.take<__nv_bfloat16>(w.vc * w.m_pad);
  w.dzT[1] = c.take<__nv_bfloat16>(w.vc * w.m_pad);
  w.dh_part = w.splits > 1 ? c.take<float>(static_cast<int64_t>(w.splits) * M * d) : nullptr;
  return w;
}
bool classic_bwd() { return opts().bwd_mode == 0; }
constexpr int kBwdDwBf16 = 1 << 8;  // internal bwd flag: dW is bf16

// ---- staged layout (fwd_stage): [fwd partials][sup_z: fp32 M x k_max][bwd region], so the
// numerators the fwd writes into the bwd's dZ^T buffer and the fwd's per-(row, tile half)
// maxima both survive until the bwd.  The fwd region sits at offset 0 as in the compact
// layout; a verify call on the same ws in between overwrites it and drops the record.
struct StageLayout { size_t off_supz, off_bwd, total; };
StageLayout stage_layout(int64_t M, int64_t d, int64_t V_local, int k_max) {
  StageLayout L{};
  Carver f(nullptr);
  carve_fwd(f, M, V_local);
  L.off_supz = rup(static_cast<int64_t>(f.off), 256);
  L.off_bwd = L.off_supz + rup(M * k_max * 4, 256);
  Carver b(nullptr);
  carve_bwd(b, M, d, V_local);
  L.total = L.off_bwd + b.off;
  return L;
}
struct StageRec {
  const void* H;
  const void* W;
  int64_t M, d, V_local, voff;
  const int32_t* sup_idx;
  int k_max, bn, n_tiles;
};
std::mutex g_stage_mu;
std::vector<std::pair<const void*, StageRec>> g_stage;  // keyed by workspace pointer
void stage_put(const void* ws, const StageRec* r) {
  std::lock_guard<std::mutex> lk(g_stage_mu);
  for (size_t i = 0; i < g_stage.size(); ++i)
    if (g_stage[i].first == ws) {
      if (r) g_stage[i].second = *r;
      else g_stage.erase(g_stage.begin() + static_cast<long>(i));
      return;
    }
  if (r) g_stage.emplace_back(ws, *r);
}
bool staged_matches(const StageRec& r, const void* H, const void* W, int64_t M, int64_t d, int64_t V_local,
                    int64_t voff, const aurora_labels_t* l) {
  return r.H == H && r.W == W && r.M == M && r.d == d && r.V_local == V_local && r.voff == voff &&
         r.sup_idx == l->sup_idx && r.k_max == l->k_max && chunk_cols(V_local, M) >= V_local;
}
bool stage_take(const void* ws, StageRec* out) {
  std::lock_guard<std::mutex> lk(g_stage_mu);
  for (size_t i = 0; i < g_stage.size(); ++i)
    if (g_stage[i].first == ws) {
      *out = g_stage[i].second;
      g_stage.erase(g_stage.begin() + static_cast<long>(i));
      return true;
    }
  return false;
}

aurora_status_t check_cfg(const aurora_loss_cfg_t* cfg, int max_k = AURORA_MAX_K) {
  if (!cfg) return AURORA_ERR_INVALID_ARG;
  if (cfg->k_accept < 1 || cfg->k_accept > max_k || cfg->k_discard < 0 || cfg->k_discard > max_k)
    return AURORA_ERR_INVALID_ARG;
  if (!(cfg->lambda_discard >= 0.f) || !std::isfinite(cfg->lambda_discard)) return AURORA_ERR_INVALID_ARG;
  if (cfg->normalize != 0 && cfg->normalize != 1) return AURORA_ERR_INVALID_ARG;
  if (cfg->discard_scope != 0 && cfg->discard_scope != 1) return AURORA_ERR_INVALID_ARG;
  if (cfg->accept_loss != 0 && cfg->accept_loss != 1) return AURORA_ERR_INVALID_ARG;
  if (!(cfg->ntp_beta >= 0.f) || !std::isfinite(cfg->ntp_beta)) return AURORA_ERR_INVALID_ARG;
  if (cfg->ntp_beta > 0.f && cfg->accept_loss != 1) return AURORA_ERR_INVALID_ARG;  // NTP pairs with RKL
  if (cfg->discard_restricted != 0 && cfg->discard_restricted != 1) return AURORA_ERR_INVALID_ARG;
  if (cfg->discard_restricted && (cfg->accept_loss != 0 || cfg->k_discard < 1)) return AURORA_ERR_INVALID_ARG;
  return AURORA_OK;
}
// F2 objectives that read the dense target row again (bit 0 RKL, bit 1 dense discard KL)
int32_t objective_of(const aurora_loss_cfg_t* cfg) {
  return (cfg->accept_loss == 1 ? 1 : 0) | (cfg->k_discard == 0 ? 2 : 0) | (cfg->discard_restricted ? 4 : 0);
}
// GEMM arguments of the F2 epilogues; c0 = first T column of the GEMM's column 0.
void set_f2_args(GemmArgs& a, const aurora_labels_t* l, int64_t c0) {
  a.T = static_cast<const uint16_t*>(l->target_logits) + c0;
  a.ldT = l->ld_target;
  a.t_vec = ((reinterpret_cast<uintptr_t>(a.T) & 15) == 0 && (l->ld_target & 7) == 0) ? 1 : 0;
  a.row_class = l->row_class;
  a.f2_rkl = (l->objective & 1) ? 1 : 0;
  a.f2_dense = (l->objective & 2) ? 1 : 0;
  a.ntp_beta = l->ntp_beta;
  a.row_lse_t = l->row_lse_t;
  a.row_aux = l->row_aux;
}
bool labels_ok(const aurora_labels_t* l, bool verify_outputs, int max_k = AURORA_MAX_K_SPARSE) {
  if (!l) return false;
  if (l->k_max < 1 || l->k_max > max_k) return false;
  if (!l->sup_idx || !l->sup_p || !l->row_H || !l->row_w || !l->row_class) return false;
  if (verify_outputs && (!l->target_argmax || !l->accepted || !l->accept_len || !l->bonus || !l->counts ||
                         !l->status))
    return false;
  return true;
}
// Library-owned side streams and events (per device, created once) for the bwd:
// dW(c) (HBM-store-bound) and dH(c) (tensor-bound) run concurrently on two side
// streams; dz(c+1) on the caller's stream waits for both (single chunk buffer).
struct SideStreams {
  cudaStream_t s[2] = {nullptr, nullptr};
  cudaEvent_t ev[160];
  bool ok = false;
};
SideStreams* side_streams() {
  static std::mutex mu;
  static SideStreams per_dev[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  SideStreams& S = per_dev[dev];
  if (!S.ok) {
    for (auto& st : S.s)
      if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    for (auto& e : S.ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    S.ok = true;
  }
  return &S;
}
bool serial_bwd() { return opts().bwd_concurrent == 0; }
// the communicator's side stream and fork / join events, created on first use
bool comm_side_ready(aurora_comm_t c) {
  if (c->side) return true;
  cudaStream_t st = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return false;
  for (auto& e : c->side_ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return false;
  c->side = st;
  return true;
}

// The comm owns a device scratch for gathered per-row data; it grows on first use
// (one cudaMalloc per size increase, never in steady state).
bool ensure_scratch(aurora_comm_t c, size_t bytes) {
  if (c->scratch_bytes >= bytes) return true;
  if (c->scratch) cudaFree(c->scratch);
  c->scratch = nullptr;
  c->scratch_bytes = 0;
  if (cudaMalloc(&c->scratch, bytes) != cudaSuccess) return false;
  c->scratch_bytes = bytes;
  return true;
}
bool gemm_shape_ok(const void* H, const void* W, int64_t M, int64_t d, int64_t V_local) {
  return H && W && M >= 1 && d >= 64 && d % 64 == 0 && V_local >= 1 && al16(H) && al16(W) &&
         M <= (int64_t(1) << 31) / 2 && V_local <= (int64_t(1) << 31) / 2;
}

// The whole backward as one persistent launch (k_bwd.cu), then the dH split reduce and
// the VP / DP collectives.
aurora_status_t bwd_fused(const void* H, const void* W, int64_t M, int64_t d, int64_t V_local, int64_t vocab_offset,
                          const aurora_labels_t* labels, const float* row_lse, const float* dloss, float* dH,
                          float* dWf, int accumulate_dW, void* ws, aurora_comm_t comm, cudaStream_t s) {
  aurora_status_t st = AURORA_OK;
  Carver c(ws);
  FusedWs w = carve_fused(c, M, d, V_local);
  const int64_t nchunks = cdiv(V_local, w.vc);
  if (nchunks > kMaxChunks) return AURORA_ERR_UNSUPPORTED;
  BwdMaps maps;
  bool ok = make_tmap_bf16(&maps.H_k, H, d, M, d, 64, BM) && make_tmap_bf16(&maps.H_mn, H, d, M, d, 64, 64) &&
            make_tmap_bf16(&maps.W_k, W, d, V_local, d, 64, BN) && make_tmap_bf16(&maps.W_mn, W, d, V_local, d, 64, 64);
  for (int b = 0; b < 2; ++b)
    ok = ok && make_tmap_bf16(&maps.Z_k[b], w.dzT[b], M, w.vc, w.m_pad, 64, BM) &&
         make_tmap_bf16(&maps.Z_mn[b], w.dzT[b], M, w.vc, w.m_pad, 64, 64);
  ok = ok && make_tmap_f32_out(&maps.O_W, dWf, d, V_local, d, 1, 0);
  ok = ok && (w.splits > 1 ? make_tmap_f32_out(&maps.O_H, w.dh_part, d, M, d, w.splits, M * d)
                           : make_tmap_f32_out(&maps.O_H, dH, d, M, d, 1, 0));
  if (!ok) return AURORA_ERR_CUDA;

  BwdArgs a{};
  a.M = M;
  a.d = d;
  a.vocab_offset = vocab_offset;
  a.sup_idx = labels->sup_idx;
  a.sup_p = labels->sup_p;
  a.k_max = labels->k_max;
  a.row_lse = row_lse;
  a.row_w = labels->row_w;
  a.dloss = dloss;
  a.dzT[0] = w.dzT[0];
  a.dzT[1] = w.dzT[1];
  a.ld_dzT = w.m_pad;
  a.accumulate_dW = (accumulate_dW & 1) ? 1 : 0;
  a.dh_m_tiles = static_cast<int32_t>(cdiv(M, BM));
  a.dh_n_tiles = static_cast<int32_t>(cdiv(d, BN));
  a.tile_counter = w.counters;
  a.dz_done = w.counters + 1;
  a.rd_done = w.counters + 1 + kMaxChunks;
  a.dh_flag = w.counters + 1 + 2 * kMaxChunks;
  int base = 0;
  auto add_seg = [&](int type, int ch) {
    BwdSeg g{};
    g.type = type;
    g.chunk = ch;
    const int64_t vc = a.vc[ch];
    if (type == BT_DZ) {
      g.m_tiles = static_cast<int32_t>(cdiv(M, BM));
      g.n_tiles = static_cast<int32_t>(cdiv(vc, BN));
      g.kb_total = static_cast<int32_t>(d / BK);
      g.kb_per_split = g.kb_total;
    } else if (type == BT_DW) {
      g.m_tiles = static_cast<int32_t>(cdiv(vc, BM));
      g.n_tiles = static_cast<int32_t>(cdiv(d, BN));
      g.kb_total = static_cast<int32_t>(cdiv(M, BK));
      g.kb_per_split = g.kb_total;
    } else {
      g.m_tiles = a.dh_m_tiles;
      g.n_tiles = a.dh_n_tiles;
      g.kb_total = static_cast<int32_t>(cdiv(vc, BK));
      g.kb_per_split = static_cast<int32_t>(cdiv(g.kb_total, w.splits));
    }
    const int count = g.m_tiles * g.n_tiles * (type == BT_DH ? w.splits : 1);
    g.base = base;
    base += count;
    if (type == BT_DZ) a.n_dz[ch] = count;
    else a.n_rd[ch] += count;
    a.seg[a.nseg++] = g;
  };
  for (int64_t ch = 0; ch < nchunks; ++ch) {
    a.c0[ch] = ch * w.vc;
    a.vc[ch] = std::min(w.vc, V_local - ch * w.vc);
  }
  for (int64_t ch = 0; ch < nchunks; ++ch) {
    add_seg(BT_DZ, static_cast<int>(ch));
    if (ch >= 1) {
      add_seg(BT_DH, static_cast<int>(ch - 1));
      add_seg(BT_DW, static_cast<int>(ch - 1));
    }
  }
  add_seg(BT_DH, static_cast<int>(nchunks - 1));
  add_seg(BT_DW, static_cast<int>(nchunks - 1));
  a.total_units = base;
  a.nchunks = static_cast<int32_t>(nchunks);

  if (cudaMemsetAsync(w.counters, 0, static_cast<size_t>(w.n_counters) * sizeof(int32_t), s) != cudaSuccess)
    return AURORA_ERR_CUDA;
  prof_begin(PH_BWD_FUSED, s);
  cudaError_t e = launch_bwd_fused(maps, a, s);
  prof_end(PH_BWD_FUSED, s);
  if (e != cudaSuccess) return AURORA_ERR_CUDA;
  if (w.splits > 1) {
    prof_begin(PH_BWD_REDUCE, s);
    e = launch_splitk_reduce(w.dh_part, w.splits, M * d, dH, 0, s);
    prof_end(PH_BWD_REDUCE, s);
    if (e != cudaSuccess) return AURORA_ERR_CUDA;
  }
  if (comm && comm->dp_x() && !(accumulate_dW & AURORA_BWD_NO_DP_REDUCE)) {  // C5: DP gradient allreduce
    prof_begin(PH_COMM, s);
    if ((st = coll_allreduce(comm, G_DP, dWf, dWf, static_cast<size_t>(V_local * d), DT_F32, s)) != AURORA_OK)
      return st;
    prof_end(PH_COMM, s);
  }
  if (comm && comm->vp_x()) {  // C4: VP dH allreduce
    prof_begin(PH_COMM, s);
    if ((st = coll_allreduce(comm, G_VP, dH, dH, static_cast<size_t>(M * d), DT_F32, s)) != AURORA_OK)
      return st;
    prof_end(PH_COMM, s);
  }
  return AURORA_OK;
}

}  // namespace
int opt_tree_bwd_split() { return opts().tree_bwd_split; }
int opt_tree_fwd_tc() { return opts().tree_fwd_tc; }
int opt_tree_bwd_tc() { return opts().tree_bwd_tc; }
int opt_dw_adamw_qe() { return opts().dw_adamw_qe; }
}  // namespace aur

using namespace aur;

extern "C" {

const char* aurora_status_string(aurora_status_t s) {
  switch (s) {
    case AURORA_OK: return "ok";
    case AURORA_ERR_INVALID_ARG: return "invalid argument";
    case AURORA_ERR_STRUCTURE: return "malformed draft tree (parents)";
    case AURORA_ERR_RANGE: return "token id out of range";
    case AURORA_ERR_NONFINITE: return "non-finite target logits";
    case AURORA_ERR_UNSUPPORTED: return "unsupported configuration";
    case AURORA_ERR_WORKSPACE: return "workspace missing or too small";
    case AURORA_ERR_CUDA: return "CUDA error";
    case AURORA_ERR_NCCL: return "NCCL error";
  }
  return "unknown status";
}

const char* aurora_build_info(void) {
  return "libaurora abi=2 target=sm_100a engine=tcgen05.mma cta_group::1 M128xN{256,224,192}xK16 / cta_group::2 "
         "M256xN256, TMA SW128 4/6-stage ring, TMEM 2x256 cols, TMA bulk-store epilogue; scan=16B ld.global.nc; "
         "objectives: Eq.3 FKL, F1 sparse top-K (k<=1024), F2 RKL+NTP / dense KL; F3 fused AdamW";
}

uint64_t aurora_launch_count(void) { return g_launches.load(); }

aurora_status_t aurora_set_option(const char* name, int64_t value) {
  if (!name) return AURORA_ERR_INVALID_ARG;
  Options& o = opts();
  if (std::strcmp(name, "gemm_pair") == 0 && value >= 0 && value <= 2) { o.gemm_pair = static_cast<int>(value); return AURORA_OK; }
  if (std::strcmp(name, "bwd_mode") == 0 && value >= 0 && value <= 1) { o.bwd_mode = static_cast<int>(value); return AURORA_OK; }
  if (std::strcmp(name, "tree_fwd_tc") == 0 && value >= 0 && value <= 3) {
    o.tree_fwd_tc = static_cast<int>(value);
    return AURORA_OK;
  }
  if (std::strcmp(name, "tree_bwd_tc") == 0 && (value == 0 || value == 1)) {
    o.tree_bwd_tc = static_cast<int>(value);
    return AURORA_OK;
  }
  if (std::strcmp(name, "tree_bwd_split") == 0 && (value == 0 || value == 1)) {
    o.tree_bwd_split = static_cast<int>(value);
    return AURORA_OK;
  }
  if (std::strcmp(name, "dw_resident") == 0 && (value == 0 || value == 1)) {
    o.dw_resident = static_cast<int>(value);
    return AURORA_OK;
  }
  if (std::strcmp(name, "scan_ctas") == 0 && value >= 1 && value <= 16) {
    o.scan_ctas = static_cast<int>(value);
    return AURORA_OK;
  }
  if (std::strcmp(name, "gram_norm") == 0 && (value == 0 || value == 1)) {
    o.gram_norm = static_cast<int>(value);
    return AURORA_OK;
  }
  if (std::strcmp(name, "debug_gemm_group") == 0 && value >= -64 && value <= 64) {
    o.debug_gemm_group = static_cast<int>(value);
    return AURORA_OK;
  }
  if (std::strcmp(name, "scan_flat") == 0 && value >= 0 && value <= 2) {
    o.scan_flat = static_cast<int>(value);
    return AURORA_OK;
  }
  if (std::strcmp(name, "scan_ring") == 0 && (value == 0 || value == 1)) {
    o.scan_ring = static_cast<int>(value);
    return AURORA_OK;
  }
  if (std::strcmp(name, "dw_adamw_qe") == 0 && value >= 0 && value <= 2) {
    o.dw_adamw_qe = static_cast<int>(value);
    return AURORA_OK;
  }
  if (std::strcmp(name, "fwd_stage") == 0 && (value == 0 || value == 1)) {
    o.fwd_stage = static_cast<int>(value);
    return AURORA_OK;
  }
  if (std::strcmp(name, "dz_chunk_bytes") == 0 && value >= 1) {
    o.dz_chunk_bytes = value;
    return AURORA_OK;
  }
  if (std::strcmp(name, "tile_n") == 0 && (value == 0 || value == 256 || value == 224 || value == 192)) {
    o.tile_n = static_cast<int>(value);
    return AURORA_OK;
  }
  if (std::strcmp(name, "bwd_concurrent") == 0 && value >= 0 && value <= 1) {
    o.bwd_concurrent = static_cast<int>(value);
    return AURORA_OK;
  }
  return AURORA_ERR_INVALID_ARG;
}

int64_t aurora_get_option(const char* name) {
  if (!name) return -1;
  const Options& o = opts();
  if (std::strcmp(name, "gemm_pair") == 0) return o.gemm_pair;
  if (std::strcmp(name, "bwd_mode") == 0) return o.bwd_mode;
  if (std::strcmp(name, "tree_bwd_split") == 0) return o.tree_bwd_split;
  if (std::strcmp(name, "tree_fwd_tc") == 0) return o.tree_fwd_tc;
  if (std::strcmp(name, "tree_bwd_tc") == 0) return o.tree_bwd_tc;
  if (std::strcmp(name, "bwd_concurrent") == 0) return o.bwd_concurrent;
  if (std::strcmp(name, "tile_n") == 0) return o.tile_n;
  if (std::strcmp(name, "dz_chunk_bytes") == 0) return o.dz_chunk_bytes;
  if (std::strcmp(name, "scan_ctas") == 0) return o.scan_ctas;
  if (std::strcmp(name, "dw_resident") == 0) return o.dw_resident;
  if (std::strcmp(name, "fwd_stage") == 0) return o.fwd_stage;
  if (std::strcmp(name, "scan_ring") == 0) return o.scan_ring;
  if (std::strcmp(name, "scan_flat") == 0) return o.scan_flat;
  if (std::strcmp(name, "dw_adamw_qe") == 0) return o.dw_adamw_qe;
  if (std::strcmp(name, "debug_gemm_group") == 0) return o.debug_gemm_group;
  if (std::strcmp(name, "gram_norm") == 0) return o.gram_norm;
  if (std::strcmp(name, "pair_max_active_clusters") == 0) return g_pair_max_clusters;
  return -1;
}

void aurora_profile_enable(int enable) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_on = enable != 0;
}

namespace {
int profile_collect(const char** names, float* total_ms, int32_t* count, int max, bool recycle) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  float tot[PH_COUNT] = {0};
  int cnt[PH_COUNT] = {0};
  for (auto& r : g_prof_done) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
      tot[r.phase] += ms;
      cnt[r.phase] += 1;
    }
    if (recycle) {
      g_ev_pool.push_back(r.a);
      g_ev_pool.push_back(r.b);
    }
  }
  if (recycle) g_prof_done.clear();
  int n = 0;
  for (int p = 0; p < PH_COUNT && n < max; ++p) {
    if (names) names[n] = kPhaseNames[p];
    if (total_ms) total_ms[n] = tot[p];
    if (count) count[n] = cnt[p];
    ++n;
  }
  return n;
}
}  // namespace

int aurora_profile_read(const char** names, float* total_ms, int32_t* count, int max) {
  return profile_collect(names, total_ms, count, max, true);
}

int aurora_profile_peek(const char** names, float* total_ms, int32_t* count, int max) {
  return profile_collect(names, total_ms, count, max, false);
}

size_t aurora_workspace_size(int op, int64_t M, int64_t d, int64_t V_local, const aurora_loss_cfg_t* cfg) {
  if (M < 1 || V_local < 1 || d < 1 || !cfg || op < 0 || op > 3) return 0;
  const int k_max = std::max(cfg->k_accept, cfg->k_discard);
  if (k_max < 1 || k_max > AURORA_MAX_K_SPARSE) return 0;
  size_t best = 0;
  if (op == AURORA_OP_VERIFY || op == AURORA_OP_ALL) {
    Carver c(nullptr);
    if (k_max <= AURORA_MAX_K) carve_verify(c, M, V_local, AURORA_MAX_K);
    else carve_verify_long(c, M, k_max);
    best = std::max(best, c.off);
  }
  if (op == AURORA_OP_FWD || op == AURORA_OP_ALL) {
    Carver c(nullptr);
    carve_fwd(c, M, V_local);
    best = std::max(best, c.off);
  }
  if (op == AURORA_OP_BWD || op == AURORA_OP_ALL) {
    Carver c(nullptr);
    carve_bwd(c, M, d, V_local);
    best = std::max(best, c.off);
    Carver f(nullptr);
    carve_fused(f, M, d, V_local);
    best = std::max(best, f.off);
  }
  if (op == AURORA_OP_ALL) best = std::max(best, stage_layout(M, d, V_local, k_max).total);  // fwd_stage
  return rup(static_cast<int64_t>(best), 256) + 256;
}

aurora_status_t aurora_verify_labels(const aurora_trace_t* t, const aurora_loss_cfg_t* cfg, aurora_labels_t* out,
                                     void* ws, size_t ws_bytes, aurora_comm_t comm, void* stream) {
  if (!t || !out) return AURORA_ERR_INVALID_ARG;
  aurora_status_t st = check_cfg(cfg);
  if (st != AURORA_OK) return st;
  if (t->R < 1 || t->N < 1 || t->N > AURORA_MAX_NODES || !t->draft_tokens || !t->target_logits) return AURORA_ERR_INVALID_ARG;
  if (t->V < 1 || t->V_local < 1 || t->vocab_offset < 0 || t->vocab_offset + t->V_local > t->V ||
      t->ld_target < t->V_local || t->V > INT32_MAX)
    return AURORA_ERR_INVALID_ARG;
  if (!labels_ok(out, true, AURORA_MAX_K)) return AURORA_ERR_INVALID_ARG;
  const int k_max = out->k_max;
  if (k_max < std::max(cfg->k_accept, cfg->k_discard)) return AURORA_ERR_INVALID_ARG;
  if (std::max(cfg->k_accept, cfg->k_discard) > t->V) return AURORA_ERR_INVALID_ARG;
  const int64_t M = static_cast<int64_t>(t->R) * (t->N + 1);
  if (!ws || ws_bytes < aurora_workspace_size(AURORA_OP_VERIFY, M, 64, t->V_local, cfg)) return AURORA_ERR_WORKSPACE;
  if (comm && comm->vp_size > 1 && t->V_local == t->V) return AURORA_ERR_INVALID_ARG;  // VP needs shards
  const int32_t objective = objective_of(cfg);
  if ((objective & 3) && (!out->row_lse_t || !out->row_aux)) return AURORA_ERR_INVALID_ARG;  // F2 row statistics
  if ((objective & 4) && (!out->row_aux || (comm && comm->vp_size > 1))) return AURORA_ERR_UNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  out->objective = objective;
  out->ntp_beta = cfg->ntp_beta;
  stage_put(ws, nullptr);  // the verify scratch overlaps a staged forward's partials

  Carver c(ws);
  VerifyWs w = carve_verify(c, M, t->V_local, k_max);
  VerifyLaunch p{};
  p.T = static_cast<const uint16_t*>(t->target_logits);
  p.ldT = t->ld_target;
  p.V_local = t->V_local;
  p.vocab_offset = t->vocab_offset;
  p.V = t->V;
  p.M = static_cast<int32_t>(M);
  p.R = t->R;
  p.N = t->N;
  p.k_max = k_max;
  p.nseg = ring_nseg(M, t->V_local);
  p.seg_len = rup(cdiv(t->V_local, p.nseg), 8);
  const bool ring = opts().scan_ring && scan_ring_ok(p);
  if (!ring) {
    p.nseg = scan_nseg(M, t->V_local);
    p.seg_len = rup(cdiv(t->V_local, p.nseg), 8);
  }
  // The flat scan removes the (row, segment) grid's wave tail; where that grid is a single partial
  // wave or its last wave is mostly full, the per-row CTAs (one shared floor and warm start per
  // row) are faster (measured: qwen3 M = 1792, 4.04 waves: flat 0.147 vs 0.166 ms; llama M = 384,
  // 0.86 waves: 0.057 vs 0.043 ms).  scan_flat = 2 forces the flat scan.
  const double seg_waves = static_cast<double>(M) * p.nseg / (3.0 * kNumSMs);
  const bool flat_pays = opts().scan_flat == 2 || (seg_waves >= 2.0 && seg_waves - std::floor(seg_waves) < 0.5);
  const bool flat = !ring && opts().scan_flat && flat_pays && scan_flat_ok(p);
  int nlists = ring ? p.nseg * scan_ring_lists() : p.nseg;
  p.draft = t->draft_tokens;
  p.parents = t->parents;
  p.num_nodes = t->num_nodes;
  p.cand_val = w.cand_val;
  p.cand_idx = w.cand_idx;
  p.top_val = w.top_val;
  p.top_idx = w.top_idx;
  p.ept = w.ept;
  p.lab = *out;
  p.cfg = *cfg;

  cudaError_t e;
  if ((e = cudaMemsetAsync(out->counts, 0, 2 * sizeof(int32_t), s)) != cudaSuccess) return AURORA_ERR_CUDA;
  if ((e = cudaMemsetAsync(out->status, 0, sizeof(uint32_t), s)) != cudaSuccess) return AURORA_ERR_CUDA;
  prof_begin(PH_SCAN, s);
  if ((e = (ring   ? launch_target_scan_ring(p, s)
             : flat ? launch_target_scan_flat(p, &nlists, s)
                    : launch_target_scan(p, s))) != cudaSuccess)
    return AURORA_ERR_CUDA;
  if ((e = launch_topk_merge(p, w.cand_val, w.cand_idx, nlists, static_cast<int64_t>(nlists) * k_max, k_max, s)) !=
      cudaSuccess)
    return AURORA_ERR_CUDA;
  prof_end(PH_SCAN, s);
  if (comm && comm->vp_x()) {
    // C1: gather every VP rank's (value-ordered) top list and merge in global order.
    const size_t per = static_cast<size_t>(M) * k_max;
    const size_t need = 2 * per * comm->vp_size * sizeof(float);
    if (!ensure_scratch(comm, need)) return AURORA_ERR_CUDA;
    float* gv = static_cast<float*>(comm->scratch);
    int32_t* gi = reinterpret_cast<int32_t*>(gv + per * comm->vp_size);
    prof_begin(PH_COMM, s);
    if ((st = coll_allgather(comm, G_VP, w.top_val, gv, per, DT_F32, s)) != AURORA_OK) return st;
    if ((st = coll_allgather(comm, G_VP, w.top_idx, gi, per, DT_I32, s)) != AURORA_OK) return st;
    prof_end(PH_COMM, s);
    // gathered layout [rank][M][k]: list l of row m at l*M*k + m*k (global ids already)
    if ((e = launch_topk_merge(p, gv, gi, comm->vp_size, k_max, static_cast<int64_t>(M) * k_max, s)) != cudaSuccess)
      return AURORA_ERR_CUDA;
  }
  if (objective & 3) {  // F2: row statistics of T (a second read of T, so it counts as scan time)
    prof_begin(PH_SCAN, s);
    if (comm && comm->vp_x()) {  // VP: per-rank (max, sum, sum*t) triples -> allgather -> merge
      p.lse_part = w.lse_part;
      if ((e = launch_row_lse_t(p, s)) != cudaSuccess) return AURORA_ERR_CUDA;
      const size_t per = static_cast<size_t>(M) * 3;
      if (!ensure_scratch(comm, per * comm->vp_size * sizeof(float))) return AURORA_ERR_CUDA;
      if ((st = coll_allgather(comm, G_VP, w.lse_part, comm->scratch, per, DT_F32, s)) != AURORA_OK) return st;
      p.lse_part = nullptr;
      if ((e = launch_row_lse_t_combine(p, static_cast<const float*>(comm->scratch), comm->vp_size, s)) !=
          cudaSuccess)
        return AURORA_ERR_CUDA;
    } else if ((e = launch_row_lse_t(p, s)) != cudaSuccess) {
      return AURORA_ERR_CUDA;
    }
    prof_end(PH_SCAN, s);
  }
  prof_begin(PH_VERIFY, s);
  if ((e = launch_verify(p, s)) != cudaSuccess) return AURORA_ERR_CUDA;
  if (comm && comm->dp_x()) {
    if ((st = coll_allreduce(comm, G_DP, out->counts, out->counts, 2, DT_I32, s)) != AURORA_OK)
      return st;
  }
  if ((e = launch_finalize(p, s)) != cudaSuccess) return AURORA_ERR_CUDA;
  prof_end(PH_VERIFY, s);
  return AURORA_OK;
}

aurora_status_t aurora_verify_labels_topk(const aurora_trace_topk_t* t, const aurora_loss_cfg_t* cfg,
                                          aurora_labels_t* out, void* ws, size_t ws_bytes, aurora_comm_t comm,
                                          void* stream) {
  if (!t || !out) return AURORA_ERR_INVALID_ARG;
  aurora_status_t st = check_cfg(cfg, AURORA_MAX_K_SPARSE);
  if (st != AURORA_OK) return st;
  if (t->R < 1 || t->N < 1 || t->N > AURORA_MAX_NODES || !t->draft_tokens || !t->target_ids || !t->target_vals)
    return AURORA_ERR_INVALID_ARG;
  if (t->V < 1 || t->V > INT32_MAX || t->K_t < 1) return AURORA_ERR_INVALID_ARG;
  if (!labels_ok(out, true)) return AURORA_ERR_INVALID_ARG;
  const int k_max = out->k_max;
  const int kk = std::max(cfg->k_accept, cfg->k_discard);
  if (k_max < kk || kk > t->K_t) return AURORA_ERR_INVALID_ARG;
  const bool long_path = kk > AURORA_MAX_K;
  if (long_path && t->K_t > AURORA_MAX_KT_SPARSE) return AURORA_ERR_UNSUPPORTED;
  if (!long_path && k_max > AURORA_MAX_K) return AURORA_ERR_INVALID_ARG;  // warp lists hold <= 16
  const int64_t M = static_cast<int64_t>(t->R) * (t->N + 1);
  if (objective_of(cfg) & 3) return AURORA_ERR_UNSUPPORTED;  // F2 RKL / dense KL need the dense target row
  if (cfg->discard_restricted && (!out->row_aux || (comm && comm->vp_size > 1))) return AURORA_ERR_UNSUPPORTED;
  if (!ws || ws_bytes < aurora_workspace_size(AURORA_OP_VERIFY, M, 64, t->K_t, cfg)) return AURORA_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  out->objective = objective_of(cfg) & 4;
  out->ntp_beta = 0.f;
  stage_put(ws, nullptr);
  Carver c(ws);
  VerifyWs w = long_path ? carve_verify_long(c, M, kk) : carve_verify(c, M, t->K_t, k_max);
  VerifyLaunch p{};
  p.V = t->V;
  p.V_local = t->V;
  p.M = static_cast<int32_t>(M);
  p.R = t->R;
  p.N = t->N;
  p.k_max = k_max;
  p.k_top = kk;
  p.nseg = 1;
  p.draft = t->draft_tokens;
  p.parents = t->parents;
  p.num_nodes = t->num_nodes;
  p.top_val = w.top_val;
  p.top_idx = w.top_idx;
  p.lab = *out;
  p.cfg = *cfg;
  if (cudaMemsetAsync(out->counts, 0, 2 * sizeof(int32_t), s) != cudaSuccess) return AURORA_ERR_CUDA;
  if (cudaMemsetAsync(out->status, 0, sizeof(uint32_t), s) != cudaSuccess) return AURORA_ERR_CUDA;
  const uint16_t* vals = static_cast<const uint16_t*>(t->target_vals);
  prof_begin(PH_SCAN, s);
  cudaError_t e = long_path ? launch_sort_pairs(p, t->target_ids, vals, t->K_t, s)
                            : launch_target_scan_topk(p, t->target_ids, vals, t->K_t, s);
  if (e != cudaSuccess) return AURORA_ERR_CUDA;
  prof_end(PH_SCAN, s);
  prof_begin(PH_VERIFY, s);
  if (launch_verify(p, s) != cudaSuccess) return AURORA_ERR_CUDA;
  if (comm && comm->dp_x()) {
    if ((st = coll_allreduce(comm, G_DP, out->counts, out->counts, 2, DT_I32, s)) != AURORA_OK)
      return st;
  }
  if ((long_path ? launch_finalize_long(p, s) : launch_finalize(p, s)) != cudaSuccess) return AURORA_ERR_CUDA;
  prof_end(PH_VERIFY, s);
  return AURORA_OK;
}

aurora_status_t aurora_spec_loss_fwd(const void* H, const void* W, int64_t M, int64_t d, int64_t V_local,
                                     int64_t vocab_offset, const aurora_labels_t* labels, float* row_lse,
                                     float* row_loss, float* loss, void* ws, size_t ws_bytes, aurora_comm_t comm,
                                     void* stream) {
  aurora_status_t st = AURORA_OK;
  if (!gemm_shape_ok(H, W, M, d, V_local) || vocab_offset < 0) return AURORA_ERR_INVALID_ARG;
  if (!labels_ok(labels, false) || !row_lse || !loss) return AURORA_ERR_INVALID_ARG;
  aurora_loss_cfg_t dummy{1, 1, 1.f, 0, 0};
  if (!ws || ws_bytes < aurora_workspace_size(AURORA_OP_FWD, M, d, V_local, &dummy)) return AURORA_ERR_WORKSPACE;
  const int32_t objective = labels->objective & 3;  // the T-reading F2 objectives
  const bool restricted = (labels->objective & 4) != 0;
  if (restricted && (!labels->row_aux || (comm && comm->vp_size > 1))) return AURORA_ERR_UNSUPPORTED;
  if (objective && (!labels->target_logits || !labels->row_lse_t || !labels->row_aux ||
                    labels->ld_target < V_local))
    return AURORA_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Carver c(ws);
  FwdWs w = carve_fwd(c, M, V_local);

  const int pf = pair_for(M);
  const int bn = kmajor_bn(cdiv(M, BM * pf), V_local, pf);
  CUtensorMap tmH, tmW;
  if (!make_tmap_bf16(&tmH, H, d, M, d, 64, BM)) return AURORA_ERR_CUDA;
  if (!make_tmap_bf16(&tmW, W, d, V_local, d, 64, bn / pf)) return AURORA_ERR_CUDA;
  GemmArgs a{};
  a.m_tiles = static_cast<int32_t>(cdiv(M, BM * pf));
  a.n_tiles = static_cast<int32_t>(cdiv(V_local, bn));
  a.splits = 1;
  a.kb_total = static_cast<int32_t>(d / BK);
  a.kb_per_split = a.kb_total;
  a.M = M;
  a.N = V_local;
  a.sup_idx = labels->sup_idx;
  a.sup_p = labels->sup_p;
  a.k_max = labels->k_max;
  a.col_gid0 = vocab_offset;
  a.p_max = w.pm;
  a.p_sum = w.ps;
  a.p_u = w.pu;
  if (objective) {
    set_f2_args(a, labels, 0);
    a.p_r = w.pr;
  }
  // Eq. 3 with the whole local vocabulary in one dZ^T chunk and a workspace holding the
  // staged layout: the epilogue also writes exp(z - m_half) into the bwd's dZ^T buffer and
  // keeps the support logits, and the bwd skips the recompute GEMM.
  const StageLayout L = stage_layout(M, d, V_local, labels->k_max);
  const bool stage = opts().fwd_stage && !objective && classic_bwd() && chunk_cols(V_local, M) >= V_local &&
                     ws_bytes >= L.total;
  if (restricted && !stage) return AURORA_ERR_UNSUPPORTED;  // needs the support logits of the staged fwd
  int epi = objective ? EPI_FWD_STATS_T : EPI_FWD_STATS;
  if (stage) {
    Carver cb(static_cast<char*>(ws) + L.off_bwd);
    BwdWs bw = carve_bwd(cb, M, d, V_local);
    a.dzT = bw.dzT;
    a.ld_dzT = bw.m_pad;
    a.sup_z = reinterpret_cast<float*>(static_cast<char*>(ws) + L.off_supz);
    epi = EPI_FWD_STAGE;
  }
  prof_begin(PH_FWD_GEMM, s);
  cudaError_t e = launch_umma_gemm(epi, false, false, tmH, tmW, a, s, nullptr, pf, bn);
  prof_end(PH_FWD_GEMM, s);
  if (e != cudaSuccess) return AURORA_ERR_CUDA;
  if (stage) {
    const StageRec rec{H, W, M, d, V_local, vocab_offset, labels->sup_idx, labels->k_max, bn, a.n_tiles};
    stage_put(ws, &rec);
  } else {
    stage_put(ws, nullptr);
  }
  prof_begin(PH_FWD_COMBINE, s);
  if ((e = launch_reduce_partials(w.pm, w.ps, w.pu, objective ? w.pr : nullptr, M, 2 * a.n_tiles, w.msu, s)) != cudaSuccess) return AURORA_ERR_CUDA;
  const float* msu_all = w.msu;
  int P = 1;
  if (comm && comm->vp_x()) {
    const size_t need = static_cast<size_t>(M) * kMsu * comm->vp_size * sizeof(float);
    if (!ensure_scratch(comm, need)) return AURORA_ERR_CUDA;
    if ((st = coll_allgather(comm, G_VP, w.msu, comm->scratch, static_cast<size_t>(M) * kMsu, DT_F32, s)) != AURORA_OK) return st;
    msu_all = static_cast<const float*>(comm->scratch);
    P = comm->vp_size;
  }
  int nb = 0;
  RowF2 f2{(objective & 1) ? 1 : 0, labels->ntp_beta, labels->row_lse_t, labels->row_aux, restricted ? 1 : 0,
           restricted ? reinterpret_cast<const float*>(static_cast<char*>(ws) + L.off_supz) : nullptr,
           labels->sup_idx, labels->k_max};
  if ((e = launch_row_combine(msu_all, P, M, labels->row_H, labels->row_w, labels->row_class, row_lse, row_loss,
                              w.bp, &nb, f2, s)) != cudaSuccess)
    return AURORA_ERR_CUDA;
  if ((e = launch_loss_sum(w.bp, nb, loss, s)) != cudaSuccess) return AURORA_ERR_CUDA;
  if (comm && comm->dp_x()) {
    if ((st = coll_allreduce(comm, G_DP, loss, loss, 1, DT_F32, s)) != AURORA_OK)
      return st;
  }
  prof_end(PH_FWD_COMBINE, s);
  return AURORA_OK;
}

// The chunked backward (dz -> dW -> dH per dZ^T chunk).  dWf == nullptr skips dW and its
// DP allreduce (the F3 fused optimizer recomputes dW tiles from the dZ^T left in ws).
// staged: the forward left exp(z - m_half) in the dZ^T buffer of the staged layout (one
// chunk): the recompute GEMM is replaced by the in-place rescale + the support fix-up.
static aurora_status_t bwd_classic_impl(const void* H, const void* W, int64_t M, int64_t d, int64_t V_local,
                                        int64_t vocab_offset, const aurora_labels_t* labels,
                                        const float* row_lse, const float* dloss, float* dH, float* dWf,
                                        int accumulate_dW, void* ws, aurora_comm_t comm, cudaStream_t s,
                                        int32_t objective, const StageRec* staged = nullptr,
                                        __nv_bfloat16** dzT_used = nullptr) {
  aurora_status_t st = AURORA_OK;
  const StageLayout SL = staged ? stage_layout(M, d, V_local, staged->k_max) : StageLayout{};
  Carver c(static_cast<char*>(ws) + (staged ? SL.off_bwd : 0));
  BwdWs w = carve_bwd(c, M, d, V_local);
  if (dzT_used) *dzT_used = w.dzT;

  CUtensorMap tmH_k, tmH_mn;
  if (!make_tmap_bf16(&tmH_k, H, d, M, d, 64, BM)) return AURORA_ERR_CUDA;
  if (!make_tmap_bf16(&tmH_mn, H, d, M, d, 64, 64)) return AURORA_ERR_CUDA;
  const int64_t nchunks = cdiv(V_local, w.vc);
  if (3 * nchunks + 1 > kCounters) return AURORA_ERR_UNSUPPORTED;
  const __nv_bfloat16* Wb = static_cast<const __nv_bfloat16*>(W);
  // Streams: dz on the caller's stream; dW and dH on two side streams (or all serial).
  SideStreams* S = serial_bwd() ? nullptr : side_streams();
  cudaStream_t sW = S ? S->s[0] : s, sH = S ? S->s[1] : s;
  cudaEvent_t* ev = S ? S->ev : nullptr;  // [0] start, [1+3c] dz(c), [2+3c] dW(c), [3+3c] dH(c)
  // Serial backward under VP: dH before dW in every chunk, and the C4 allreduce of dH on the
  // comm's own side stream while the last chunk's dW GEMM runs (dW needs no communication)
  // (not when a DP allreduce of dW follows on the main stream: two collectives of different
  // communicators in flight at once could be ordered differently on different GPUs)
  const bool dp_c5 = comm && comm->dp_x() && dWf && !(accumulate_dW & AURORA_BWD_NO_DP_REDUCE);
  const bool c4_side = !S && comm && comm->vp_x() && !dp_c5 && dWf && comm_side_ready(comm);
  if (cudaMemsetAsync(w.counters, 0, kCounters * sizeof(int32_t), s) != cudaSuccess) return AURORA_ERR_CUDA;
  if (S) {
    if (cudaEventRecord(ev[0], s) != cudaSuccess) return AURORA_ERR_CUDA;
    cudaStreamWaitEvent(sW, ev[0], 0);
    cudaStreamWaitEvent(sH, ev[0], 0);
  }
  for (int64_t ch = 0; ch < nchunks; ++ch) {
    const int64_t c0 = ch * w.vc;
    const int64_t vc = std::min(w.vc, V_local - c0);
    __nv_bfloat16* dzT = w.dzT;
    const int pz = pair_for(M), pw = pair_for(vc);
    const int bz = kmajor_bn(cdiv(M, BM * pz), vc, pz);
    CUtensorMap tmW_k, tmW_mn, tmZ_k, tmZ_mn;
    if (!make_tmap_bf16(&tmW_k, Wb + c0 * d, d, vc, d, 64, bz / pz)) return AURORA_ERR_CUDA;
    if (!make_tmap_bf16(&tmW_mn, Wb + c0 * d, d, vc, d, 64, 64)) return AURORA_ERR_CUDA;
    if (!make_tmap_bf16(&tmZ_k, dzT, M, vc, w.m_pad, 64, BM)) return AURORA_ERR_CUDA;
    if (!make_tmap_bf16(&tmZ_mn, dzT, M, vc, w.m_pad, 64, 64)) return AURORA_ERR_CUDA;
    if (S && ch >= 1) {  // dz(ch) overwrites the chunk buffer read by dW(ch-1), dH(ch-1)
      cudaStreamWaitEvent(s, ev[2 + 3 * (ch - 1)], 0);
      cudaStreamWaitEvent(s, ev[3 + 3 * (ch - 1)], 0);
    }

    // A7: recompute Z tiles, dz -> dZ^T chunk (bf16)
    GemmArgs a{};
    a.m_tiles = static_cast<int32_t>(cdiv(M, BM * pz));
    a.n_tiles = static_cast<int32_t>(cdiv(vc, bz));
    a.splits = 1;
    a.kb_total = static_cast<int32_t>(d / BK);
    a.kb_per_split = a.kb_total;
    a.M = M;
    a.N = vc;
    a.sup_idx = labels->sup_idx;
    a.sup_p = labels->sup_p;
    a.k_max = labels->k_max;
    a.col_gid0 = vocab_offset + c0;
    a.row_lse = row_lse;
    a.row_w = labels->row_w;
    a.dloss = dloss;
    a.dzT = dzT;
    a.ld_dzT = w.m_pad;
    a.tile_counter = w.counters + 3 * ch;
    if (objective) set_f2_args(a, labels, c0);
    cudaError_t e;
    if (staged) {
      Carver fc(ws);
      const FwdWs fw = carve_fwd(fc, M, V_local);
      prof_begin(PH_BWD_RESCALE, s);
      const int restricted = (labels->objective & 4) ? 1 : 0;  // F2 restricted-softmax DISCARD rows
      e = launch_dz_rescale(dzT, w.m_pad, M, V_local, staged->bn, staged->n_tiles, fw.pm, row_lse, labels->row_w, dloss,
                            labels->row_class, restricted, s);
      if (e == cudaSuccess)
        e = launch_dz_support_fix(dzT, w.m_pad, M, V_local, vocab_offset, labels,
                                  reinterpret_cast<const float*>(static_cast<char*>(ws) + SL.off_supz), row_lse, dloss,
                                  restricted, s);
      prof_end(PH_BWD_RESCALE, s);
    } else {
      prof_begin(PH_BWD_DZ, s);
      e = launch_umma_gemm(objective ? EPI_BWD_DZ_T : EPI_BWD_DZ, false, false, tmH_k, tmW_k, a, s, nullptr, pz, bz);
      prof_end(PH_BWD_DZ, s);
    }
    if (e != cudaSuccess) return AURORA_ERR_CUDA;
    if (S) {
      cudaEventRecord(ev[1 + 3 * ch], s);
      cudaStreamWaitEvent(sW, ev[1 + 3 * ch], 0);
      cudaStreamWaitEvent(sH, ev[1 + 3 * ch], 0);
    }

    // A9: dH += dZ W[chunk]   (A = dZ^T as MN-major, B = W MN-major, K = vc)
    GemmArgs h{};
    const int ph = pair_for(M);
    h.m_tiles = static_cast<int32_t>(cdiv(M, BM * ph));
    h.n_tiles = static_cast<int32_t>(cdiv(d, BN));
    h.kb_total = static_cast<int32_t>(cdiv(vc, BK));
    h.splits = std::min<int>(dh_splits(M, d, h.kb_total, ph), w.splits);
    h.kb_per_split = static_cast<int32_t>(cdiv(h.kb_total, h.splits));
    h.splits = static_cast<int32_t>(cdiv(h.kb_total, h.kb_per_split));
    h.M = M;
    h.N = d;
    h.ld_out = d;
    h.tile_counter = w.counters + 3 * ch + 2;
    if (h.splits > 1) {
      h.out = w.dh_part;
      h.split_stride = M * d;
      h.accumulate = 0;
    } else {
      h.out = dH;
      h.accumulate = ch > 0 ? 1 : 0;
    }
    CUtensorMap tmOH;
    const bool oh = h.splits > 1 ? make_tmap_f32_out(&tmOH, w.dh_part, d, M, d, h.splits, M * d)
                                 : make_tmap_f32_out(&tmOH, dH, d, M, d, 1, 0);
    prof_begin(PH_BWD_DH, sH);
    e = launch_umma_gemm(EPI_STORE_F32, true, true, tmZ_mn, tmW_mn, h, sH, oh ? &tmOH : nullptr, ph);
    prof_end(PH_BWD_DH, sH);
    if (e != cudaSuccess) return AURORA_ERR_CUDA;
    if (h.splits > 1) {
      prof_begin(PH_BWD_REDUCE, sH);
      e = launch_splitk_reduce(w.dh_part, h.splits, M * d, dH, ch > 0 ? 1 : 0, sH);
      prof_end(PH_BWD_REDUCE, sH);
      if (e != cudaSuccess) return AURORA_ERR_CUDA;
    }
    if (S) cudaEventRecord(ev[3 + 3 * ch], sH);
    if (c4_side && ch == nchunks - 1) {  // C4 on the comm's side stream, overlapped with the last dW
      cudaEventRecord(comm->side_ev[0], s);
      cudaStreamWaitEvent(comm->side, comm->side_ev[0], 0);
      prof_begin(PH_COMM, comm->side);
      if ((st = coll_allreduce(comm, G_VP, dH, dH, static_cast<size_t>(M * d), DT_F32, comm->side)) != AURORA_OK)
        return st;
      prof_end(PH_COMM, comm->side);
      cudaEventRecord(comm->side_ev[1], comm->side);
    }
    if (dWf) {
      // A8: dW[chunk] = dZ^T H   (A = dZ^T K-major, B = H MN-major, K = M)
      GemmArgs b{};
      b.m_tiles = static_cast<int32_t>(cdiv(vc, BM * pw));
      b.n_tiles = static_cast<int32_t>(cdiv(d, BN));
      b.splits = 1;
      b.kb_total = static_cast<int32_t>(cdiv(M, BK));
      b.kb_per_split = b.kb_total;
      b.M = vc;
      b.N = d;
      b.out = dWf + c0 * d;
      b.ld_out = d;
      b.accumulate = (accumulate_dW & 1) ? 1 : 0;
      b.tile_counter = w.counters + 3 * ch + 1;
      b.n_fastest = 1;  // A = dZ^T chunk (M x vc, may exceed L2) streams once; H (B) stays in L2
      CUtensorMap tmOW;
      const bool dw_bf16 = (accumulate_dW & kBwdDwBf16) != 0;  // bf16 dW (§8(b) dW_is_bf16)
      const bool ow = dw_bf16 ? make_tmap_bf16_out(&tmOW, reinterpret_cast<uint16_t*>(dWf) + c0 * d, d, vc, d)
                              : make_tmap_f32_out(&tmOW, dWf + c0 * d, d, vc, d, 1, 0);
      prof_begin(PH_BWD_DW, sW);
      if (dw_bf16) {
        if (!ow) return AURORA_ERR_CUDA;
        e = launch_umma_gemm(EPI_STORE_BF16, false, true, tmZ_k, tmH_mn, b, sW, &tmOW, pw);
      } else if (pw == 2 && ow && opts().dw_resident && dw_resident_ok(b.kb_total))
        e = launch_dw_resident(tmZ_k, tmH_mn, tmOW, b, sW);  // small M: dZ^T rows stay in smem
      else
        e = launch_umma_gemm(EPI_STORE_F32, false, true, tmZ_k, tmH_mn, b, sW, ow ? &tmOW : nullptr, pw);
      prof_end(PH_BWD_DW, sW);
      if (e != cudaSuccess) return AURORA_ERR_CUDA;
      if (comm && comm->dp_x() && !(accumulate_dW & AURORA_BWD_NO_DP_REDUCE)) {  // C5: DP gradient allreduce of this dW chunk
        prof_begin(PH_COMM, sW);
        if ((st = coll_allreduce(comm, G_DP, dWf + c0 * d, dWf + c0 * d, static_cast<size_t>(vc * d), DT_F32, sW)) != AURORA_OK)
      return st;
        prof_end(PH_COMM, sW);
      }
      if (S) cudaEventRecord(ev[2 + 3 * ch], sW);
    }
  }
  if (S) {  // join
    cudaStreamWaitEvent(s, ev[2 + 3 * (nchunks - 1)], 0);
    cudaStreamWaitEvent(s, ev[3 + 3 * (nchunks - 1)], 0);
  }
  if (c4_side) {
    cudaStreamWaitEvent(s, comm->side_ev[1], 0);
  } else if (comm && comm->vp_x()) {  // C4: VP dH allreduce
    prof_begin(PH_COMM, s);
    if ((st = coll_allreduce(comm, G_VP, dH, dH, static_cast<size_t>(M * d), DT_F32, s)) != AURORA_OK)
      return st;
    prof_end(PH_COMM, s);
  }
  return AURORA_OK;
}

aurora_status_t aurora_spec_loss_bwd(const void* H, const void* W, int64_t M, int64_t d, int64_t V_local,
                                     int64_t vocab_offset, const aurora_labels_t* labels, const float* row_lse,
                                     const float* dloss, float* dH, void* dW, int dW_is_bf16, int accumulate_dW,
                                     void* ws, size_t ws_bytes, aurora_comm_t comm, void* stream) {
  if (!gemm_shape_ok(H, W, M, d, V_local) || vocab_offset < 0) return AURORA_ERR_INVALID_ARG;
  if (!labels_ok(labels, false) || !row_lse || !dH || !dW || !al16(dH) || !al16(dW)) return AURORA_ERR_INVALID_ARG;
  // bf16 dW: a plain TMA bf16-store epilogue; not with accumulation, a DP reduction or the
  // opt-in fused persistent backward (fp32 sums)
  if (dW_is_bf16 && ((accumulate_dW & AURORA_BWD_ACCUMULATE) || (comm && comm->dp_size > 1 &&
                                                                 !(accumulate_dW & AURORA_BWD_NO_DP_REDUCE)) ||
                     !classic_bwd()))
    return AURORA_ERR_UNSUPPORTED;
  if (dW_is_bf16) accumulate_dW |= kBwdDwBf16;
  aurora_loss_cfg_t dummy{1, 1, 1.f, 0, 0};
  if (!ws || ws_bytes < aurora_workspace_size(AURORA_OP_BWD, M, d, V_local, &dummy)) return AURORA_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  float* dWf = static_cast<float*>(dW);
  const int32_t objective = labels->objective & 3;  // the T-reading F2 objectives
  const bool restricted = (labels->objective & 4) != 0;
  if (objective && (!labels->target_logits || !labels->row_lse_t || !labels->row_aux ||
                    labels->ld_target < V_local))
    return AURORA_ERR_INVALID_ARG;
  StageRec rec;
  const bool staged = stage_take(ws, &rec) && staged_matches(rec, H, W, M, d, V_local, vocab_offset, labels) &&
                      !objective && classic_bwd() && ws_bytes >= stage_layout(M, d, V_local, rec.k_max).total;
  if (restricted && !staged) return AURORA_ERR_UNSUPPORTED;  // the support logits live in the staged ws
  // the fused persistent bwd implements Eq. 3 only; the F2 objectives take the chunked path
  if (!classic_bwd() && !objective) return bwd_fused(H, W, M, d, V_local, vocab_offset, labels, row_lse, dloss, dH, dWf,
                                       accumulate_dW, ws, comm, s);
  return bwd_classic_impl(H, W, M, d, V_local, vocab_offset, labels, row_lse, dloss, dH, dWf, accumulate_dW, ws,
                          comm, s, objective, staged ? &rec : nullptr);
}

// ---- F3 optimizer workspace: [scalars: norm^2 at 0, k_adamw_prep's sc at 16.., the int64
// device step counter at byte 128] [norm partials] [sharded mode: dW shard f32, bf16 shard]
namespace {
struct OptWs {
  float* norm_sq;
  float* sc;
  int64_t* step_dev;
  float* partials;
  float* dw_shard;
  uint16_t* wb_shard;
};
int64_t opt_parts(int64_t n) { return std::max<int64_t>(adamw_partials(), n / 4096 + 4 * 1024); }
OptWs carve_opt(Carver& c, int64_t n, int64_t shard) {
  OptWs w{};
  float* scal = c.take<float>(64);
  w.norm_sq = scal;
  w.sc = scal ? scal + 16 : nullptr;
  w.step_dev = scal ? reinterpret_cast<int64_t*>(scal + 32) : nullptr;
  w.partials = c.take<float>(opt_parts(n));
  if (shard > 0) {
    w.dw_shard = c.take<float>(shard);
    w.wb_shard = c.take<uint16_t>(shard);
  }
  return w;
}
bool adamw_cfg_ok(const aurora_adamw_cfg_t* cfg) {
  return cfg && cfg->lr >= 0.f && cfg->beta1 >= 0.f && cfg->beta1 < 1.f && cfg->beta2 >= 0.f && cfg->beta2 < 1.f &&
         cfg->eps > 0.f && cfg->weight_decay >= 0.f && std::isfinite(cfg->max_grad_norm) && cfg->warmup_steps >= 0;
}
AdamwHyper hyper_of(const aurora_adamw_cfg_t* cfg) {
  return AdamwHyper{cfg->lr, cfg->beta1, cfg->beta2, cfg->eps, cfg->weight_decay, cfg->max_grad_norm,
                    cfg->warmup_steps};
}
}  // namespace

size_t aurora_adamw_workspace_size(int64_t n) {
  if (n < 1) return 0;
  Carver c(nullptr);
  carve_opt(c, n, 0);
  return rup(static_cast<int64_t>(c.off), 256) + 256;
}

size_t aurora_adamw_sharded_workspace_size(int64_t n, int dp_size) {
  if (n < 1 || dp_size < 1) return 0;
  Carver c(nullptr);
  carve_opt(c, n, cdiv(n, dp_size));
  return rup(static_cast<int64_t>(c.off), 256) + 256;
}

aurora_status_t aurora_adamw_step(float* W_master, void* W_bf16, float* m, float* v, const float* dW, int64_t n,
                                  int64_t step, const aurora_adamw_cfg_t* cfg, const float* extra_sq, float* grad_norm,
                                  void* ws, size_t ws_bytes, aurora_comm_t comm, void* stream) {
  aurora_status_t st = AURORA_OK;
  if (!W_master || !m || !v || !dW || !cfg || n < 4 || n % 4 || step < 0) return AURORA_ERR_INVALID_ARG;
  if (!al16(W_master) || !al16(m) || !al16(v) || !al16(dW) || (W_bf16 && (reinterpret_cast<uintptr_t>(W_bf16) & 7)))
    return AURORA_ERR_INVALID_ARG;
  if (!adamw_cfg_ok(cfg)) return AURORA_ERR_INVALID_ARG;
  if (!ws || ws_bytes < aurora_adamw_workspace_size(n)) return AURORA_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Carver c(ws);
  OptWs w = carve_opt(c, n, 0);
  prof_begin(PH_OPTIM, s);
  if (launch_sumsq(dW, n, w.partials, w.norm_sq, s) != cudaSuccess) return AURORA_ERR_CUDA;
  if (comm && comm->vp_x()) {  // disjoint vocab shards: the global norm^2 sums over the VP group
    if ((st = coll_allreduce(comm, G_VP, w.norm_sq, w.norm_sq, 1, DT_F32, s)) != AURORA_OK) return st;
  }
  if (launch_adamw_prep(w.norm_sq, extra_sq, hyper_of(cfg), step, w.step_dev, w.sc, grad_norm, s) != cudaSuccess)
    return AURORA_ERR_CUDA;
  if (launch_adamw(W_master, W_bf16, m, v, dW, n, w.sc, s) != cudaSuccess) return AURORA_ERR_CUDA;
  prof_end(PH_OPTIM, s);
  return AURORA_OK;
}

aurora_status_t aurora_adamw_step_sharded(float* W_master_shard, void* W_bf16, float* m_shard, float* v_shard,
                                          const float* dW, int64_t n, int64_t step, const aurora_adamw_cfg_t* cfg,
                                          const float* extra_sq, float* grad_norm, void* ws, size_t ws_bytes,
                                          aurora_comm_t comm, void* stream) {
  aurora_status_t st = AURORA_OK;
  if (!comm || !W_master_shard || !W_bf16 || !m_shard || !v_shard || !dW || !cfg || step < 0)
    return AURORA_ERR_INVALID_ARG;
  const int P = comm->dp_size, q = comm->dp_rank;
  if (n < 4 * P || n % (4 * P)) return AURORA_ERR_INVALID_ARG;
  if (!al16(W_master_shard) || !al16(m_shard) || !al16(v_shard) || !al16(dW) || !al16(W_bf16))
    return AURORA_ERR_INVALID_ARG;
  if (!adamw_cfg_ok(cfg)) return AURORA_ERR_INVALID_ARG;
  if (!ws || ws_bytes < aurora_adamw_sharded_workspace_size(n, P)) return AURORA_ERR_WORKSPACE;
  const int64_t sh = n / P;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Carver c(ws);
  OptWs w = carve_opt(c, n, sh);
  prof_begin(PH_OPTIM, s);
  // C5': reduce-scatter of dW over the DP group (rank q receives the summed shard q)
  if (comm->dp_x()) {
    if ((st = coll_reduce_scatter(comm, G_DP, dW, w.dw_shard, static_cast<size_t>(sh), DT_F32, s)) != AURORA_OK)
      return st;
  } else if (cudaMemcpyAsync(w.dw_shard, dW, sh * sizeof(float), cudaMemcpyDeviceToDevice, s) != cudaSuccess) {
    return AURORA_ERR_CUDA;
  }
  if (launch_sumsq(w.dw_shard, sh, w.partials, w.norm_sq, s) != cudaSuccess) return AURORA_ERR_CUDA;
  // the shards are disjoint over DP (reduce-scatter slots) and over VP (vocab slices)
  if (comm->dp_x() && (st = coll_allreduce(comm, G_DP, w.norm_sq, w.norm_sq, 1, DT_F32, s)) != AURORA_OK) return st;
  if (comm->vp_size > 1 && (st = coll_allreduce(comm, G_VP, w.norm_sq, w.norm_sq, 1, DT_F32, s)) != AURORA_OK)
    return st;
  if (launch_adamw_prep(w.norm_sq, extra_sq, hyper_of(cfg), step, w.step_dev, w.sc, grad_norm, s) != cudaSuccess)
    return AURORA_ERR_CUDA;
  if (launch_adamw(W_master_shard, w.wb_shard, m_shard, v_shard, w.dw_shard, sh, w.sc, s) != cudaSuccess)
    return AURORA_ERR_CUDA;
  // every rank needs the whole updated bf16 lm_head for the next step's GEMMs
  if (comm->dp_x()) {
    if ((st = coll_allgather(comm, G_DP, w.wb_shard, W_bf16, static_cast<size_t>(sh / 2), DT_I32, s)) != AURORA_OK)
      return st;
  } else if (cudaMemcpyAsync(static_cast<uint16_t*>(W_bf16) + q * sh, w.wb_shard, sh * 2, cudaMemcpyDeviceToDevice,
                             s) != cudaSuccess) {
    return AURORA_ERR_CUDA;
  }
  prof_end(PH_OPTIM, s);
  return AURORA_OK;
}

aurora_status_t aurora_spec_loss_bwd_adamw(const void* H, void* W, int64_t M, int64_t d, int64_t V_local,
                                           int64_t vocab_offset, const aurora_labels_t* labels, const float* row_lse,
                                           const float* dloss, float* dH, float* W_master, float* m, float* v,
                                           int64_t step, const aurora_adamw_cfg_t* cfg, const float* extra_sq,
                                           float* grad_norm, void* ws, size_t ws_bytes, void* opt_ws,
                                           size_t opt_ws_bytes, aurora_comm_t comm, void* stream) {
  aurora_status_t st = AURORA_OK;
  if (!gemm_shape_ok(H, W, M, d, V_local) || vocab_offset < 0) return AURORA_ERR_INVALID_ARG;
  if (!labels_ok(labels, false) || !row_lse || !dH || !al16(dH)) return AURORA_ERR_INVALID_ARG;
  if (!W_master || !m || !v || !al16(W_master) || !al16(m) || !al16(v) || step < 0 || !adamw_cfg_ok(cfg))
    return AURORA_ERR_INVALID_ARG;
  aurora_loss_cfg_t dummy{1, 1, 1.f, 0, 0};
  if (!ws || ws_bytes < aurora_workspace_size(AURORA_OP_BWD, M, d, V_local, &dummy)) return AURORA_ERR_WORKSPACE;
  if (!opt_ws || opt_ws_bytes < aurora_adamw_workspace_size(V_local * d)) return AURORA_ERR_WORKSPACE;
  const int32_t objective = labels->objective & 3;
  const bool restricted = (labels->objective & 4) != 0;
  if (objective && (!labels->target_logits || !labels->row_lse_t || !labels->row_aux ||
                    labels->ld_target < V_local))
    return AURORA_ERR_INVALID_ARG;
  if (comm && comm->dp_size > 1) return AURORA_ERR_UNSUPPORTED;   // DP: reduce-scatter + aurora_adamw_step_sharded
  if (chunk_cols(V_local, M) < V_local) return AURORA_ERR_UNSUPPORTED;  // dZ^T of the whole slice in ws
  if (!dw_adamw_supported(V_local, d)) return AURORA_ERR_UNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // 1) dz (whole local vocabulary) and dH, no dW
  StageRec rec;
  const bool staged = stage_take(ws, &rec) && staged_matches(rec, H, W, M, d, V_local, vocab_offset, labels) &&
                      !objective && ws_bytes >= stage_layout(M, d, V_local, rec.k_max).total;
  if (restricted && !staged) return AURORA_ERR_UNSUPPORTED;
  __nv_bfloat16* dzT = nullptr;
  st = bwd_classic_impl(H, W, M, d, V_local, vocab_offset, labels, row_lse, dloss, dH, nullptr, 0, ws, comm, s,
                        objective, staged ? &rec : nullptr, &dzT);
  if (st != AURORA_OK) return st;
  // 2) dW tiles recomputed from the dZ^T left in ws: pass 1 their sum of squares (global
  //    norm), pass 2 the AdamW update from the TMEM accumulators -- dW never reaches HBM
  Carver c(nullptr);
  BwdWs w = carve_bwd(c, M, d, V_local);
  w.dzT = dzT;
  CUtensorMap tmZ_k, tmH_mn;
  if (!make_tmap_bf16(&tmZ_k, w.dzT, M, V_local, w.m_pad, 64, BM)) return AURORA_ERR_CUDA;
  if (!make_tmap_bf16(&tmH_mn, H, d, M, d, 64, 64)) return AURORA_ERR_CUDA;
  const int pw = pair_for(w.vc);
  GemmArgs b{};
  b.m_tiles = static_cast<int32_t>(cdiv(V_local, BM * pw));
  b.n_tiles = static_cast<int32_t>(cdiv(d, BN));
  b.splits = 1;
  b.kb_total = static_cast<int32_t>(cdiv(M, BK));
  b.kb_per_split = b.kb_total;
  b.M = V_local;
  b.N = d;
  b.ld_out = d;
  b.n_fastest = 1;
  const int64_t nparts = static_cast<int64_t>(b.m_tiles) * b.n_tiles * pw * kEpiWarps;
  Carver oc(opt_ws);
  OptWs ow = carve_opt(oc, V_local * d, 0);
  if (nparts > opt_parts(V_local * d)) return AURORA_ERR_WORKSPACE;
  prof_begin(PH_OPTIM, s);
  // Global norm.  Small M: the Gram form ||dZ^T H||_F^2 = sum_{m,m'} (dZ dZ^T)_{mm'} (H H^T)_{mm'}
  // (two M x M GEMMs, 2 M^2 (V + d) flops instead of the 2 M V d of recomputing every dW tile),
  // in scratch that is free at this point (the staged forward's partials, or the space after the
  // recompute layout's bwd region); otherwise the dW recompute with a sum-of-squares epilogue.
  const int64_t MM = M * M;
  char* gbase = nullptr;
  size_t gbytes = 0;
  if (staged) {
    gbase = static_cast<char*>(ws);
    gbytes = stage_layout(M, d, V_local, rec.k_max).off_supz;
  } else {
    Carver bc(nullptr);
    carve_bwd(bc, M, d, V_local);
    const size_t used = static_cast<size_t>(rup(static_cast<int64_t>(bc.off), 256));
    gbase = static_cast<char*>(ws) + used;
    gbytes = ws_bytes > used ? ws_bytes - used : 0;
  }
  int gs = 0;  // split-K factor of dZ dZ^T (K = V_local)
  if (M <= 2048 && MM % 4 == 0 && opts().gram_norm)
    for (int sp = 8; sp >= 1; --sp)
      if (static_cast<size_t>(2 + sp) * MM * 4 + 4096 <= gbytes) { gs = sp; break; }
  if (gs > 0) {
    float* Gz = reinterpret_cast<float*>(gbase);
    float* Gh = Gz + MM;
    float* gpart = Gh + MM;
    CUtensorMap tzA, tzB, tzC, thA, thB, thC;
    bool ok = make_tmap_bf16(&tzA, dzT, M, V_local, w.m_pad, 64, 64) && make_tmap_bf16(&tzB, dzT, M, V_local, w.m_pad, 64, 64);
    ok = ok && make_tmap_bf16(&thA, H, d, M, d, 64, BM) && make_tmap_bf16(&thB, H, d, M, d, 64, BN);
    GemmArgs gz{};
    gz.m_tiles = static_cast<int32_t>(cdiv(M, BM));
    gz.n_tiles = static_cast<int32_t>(cdiv(M, BN));
    gz.kb_total = static_cast<int32_t>(cdiv(V_local, BK));
    gz.kb_per_split = static_cast<int32_t>(cdiv(gz.kb_total, gs));
    gz.splits = static_cast<int32_t>(cdiv(gz.kb_total, gz.kb_per_split));
    gz.M = M;
    gz.N = M;
    gz.out = gpart;
    gz.ld_out = M;
    gz.split_stride = MM;
    ok = ok && make_tmap_f32_out(&tzC, gpart, M, M, M, gz.splits, MM);
    GemmArgs gh{};
    gh.m_tiles = gz.m_tiles;
    gh.n_tiles = gz.n_tiles;
    gh.kb_total = static_cast<int32_t>(d / BK);
    gh.kb_per_split = gh.kb_total;
    gh.splits = 1;
    gh.M = M;
    gh.N = M;
    gh.out = Gh;
    gh.ld_out = M;
    ok = ok && make_tmap_f32_out(&thC, Gh, M, M, M, 1, 0);
    if (!ok) return AURORA_ERR_CUDA;
    if (launch_umma_gemm(EPI_STORE_F32, true, true, tzA, tzB, gz, s, &tzC, 1) != cudaSuccess ||
        launch_splitk_reduce(gpart, gz.splits, MM, Gz, 0, s) != cudaSuccess ||
        launch_umma_gemm(EPI_STORE_F32, false, false, thA, thB, gh, s, &thC, 1) != cudaSuccess ||
        launch_dot(Gz, Gh, MM, ow.partials, ow.norm_sq, s) != cudaSuccess)
      return AURORA_ERR_CUDA;
  } else {
    b.out = ow.partials;
    if (launch_umma_gemm(EPI_SUMSQ, false, true, tmZ_k, tmH_mn, b, s, nullptr, pw) != cudaSuccess)
      return AURORA_ERR_CUDA;
    if (launch_sum_partials(ow.partials, static_cast<int>(nparts), ow.norm_sq, s) != cudaSuccess)
      return AURORA_ERR_CUDA;
  }
  if (comm && comm->vp_x()) {
    if ((st = coll_allreduce(comm, G_VP, ow.norm_sq, ow.norm_sq, 1, DT_F32, s)) != AURORA_OK) return st;
  }
  if (launch_adamw_prep(ow.norm_sq, extra_sq, hyper_of(cfg), step, ow.step_dev, ow.sc, grad_norm, s) != cudaSuccess)
    return AURORA_ERR_CUDA;
  if (launch_dw_adamw(w.dzT, w.m_pad, H, M, d, V_local, W_master, m, v, W, ow.sc, s) != cudaSuccess)
    return AURORA_ERR_CUDA;
  prof_end(PH_OPTIM, s);
  return AURORA_OK;
}

aurora_status_t aurora_debug_gemm(int a_mn, int b_mn, const void* A, const void* B, float* D, int64_t M, int64_t N,
                                  int64_t K, int64_t lda, int64_t ldb, int64_t ldd, void* stream) {
  if (!A || !B || !D || M < 1 || N < 1 || K < 1 || !al16(A) || !al16(B) || (lda * 2) % 16 || (ldb * 2) % 16)
    return AURORA_ERR_INVALID_ARG;
  if (ldd < N || lda < (a_mn ? M : K) || ldb < (b_mn ? N : K)) return AURORA_ERR_INVALID_ARG;
  const int pr = pair_for(M);
  CUtensorMap ta, tb;
  bool ok = a_mn ? make_tmap_bf16(&ta, A, M, K, lda, 64, 64) : make_tmap_bf16(&ta, A, K, M, lda, 64, BM);
  ok = ok && (b_mn ? make_tmap_bf16(&tb, B, N, K, ldb, 64, 64) : make_tmap_bf16(&tb, B, K, N, ldb, 64, BN / pr));
  if (!ok) return AURORA_ERR_CUDA;
  GemmArgs g{};
  static const int dbg_nfast = [] {  // diagnostics: tile raster of the test hook
    const char* e = getenv("AURORA_DBG_NFAST");
    return (e && e[0] == '1') ? 1 : 0;
  }();
  g.n_fastest = dbg_nfast;
  if (opts().debug_gemm_group) {  // test hook: the grouped raster of the F4 projections
    g.group = std::abs(opts().debug_gemm_group);
    g.group_on_n = opts().debug_gemm_group < 0 ? 1 : 0;
  }
  g.m_tiles = static_cast<int32_t>(cdiv(M, BM * pr));
  g.n_tiles = static_cast<int32_t>(cdiv(N, BN));
  g.splits = 1;
  g.kb_total = static_cast<int32_t>(cdiv(K, BK));
  g.kb_per_split = g.kb_total;
  g.M = M;
  g.N = N;
  g.out = D;
  g.ld_out = ldd;
  CUtensorMap tc;
  const bool oc = make_tmap_f32_out(&tc, D, N, M, ldd, 1, 0);
  return cuda_status(launch_umma_gemm(EPI_STORE_F32, a_mn != 0, b_mn != 0, ta, tb, g,
                                      static_cast<cudaStream_t>(stream), oc ? &tc : nullptr, pr));
}

aurora_status_t aurora_debug_dlogits_rows(const void* H, const void* W, int64_t M, int64_t d, int64_t V_local,
                                          int64_t vocab_offset, const aurora_labels_t* labels, const float* row_lse,
                                          const float* dloss, const int32_t* rows, int32_t n_rows, float* out,
                                          void* stream) {
  if (!H || !W || !labels || !row_lse || !rows || !out || n_rows < 1 || n_rows > 65535 || M < 1 || d < 1 ||
      V_local < 1)
    return AURORA_ERR_INVALID_ARG;
  return cuda_status(launch_debug_dlogits(static_cast<const __nv_bfloat16*>(H), static_cast<const __nv_bfloat16*>(W),
                                          M, d, V_local, vocab_offset, labels, row_lse, dloss, rows, n_rows, out,
                                          static_cast<cudaStream_t>(stream)));
}

}  // extern "C"

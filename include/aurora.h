/*
 * aurora.h — C-ABI boundary of the B200-native Aurora speculator-training hot path.
 *
 * Paper: "When RL Meets Adaptive Speculative Training: A Unified Training–Serving
 * System" (arXiv 2602.06932).  Citations: P:n = PAPER.md line n, S:n = SPEC.md line n.
 *
 * One trace batch (R requests x N draft nodes, M = R*(N+1) rows) goes through
 *   aurora_verify_labels  greedy verification + per-row targets
 *   aurora_spec_loss_fwd  lm_head GEMM + vocab-wide log-softmax + Eq. 3 loss
 *   aurora_spec_loss_bwd  dLogits (tiles only) -> dW_lmhead, dHidden
 * The [M x V] logits are never stored; dLogits exist only as a bf16 per-vocab-chunk
 * workspace bounded by the "dz_chunk_bytes" option (default 16 GiB; see aurora_set_option).
 *
 * Conventions (all entry points):
 *  - Pointers marked (dev) are CUDA device pointers, (host) are host pointers.  The
 *    caller owns every buffer; the library never allocates device memory on the hot
 *    path (scratch comes from `ws`, sized by aurora_workspace_size).
 *  - `stream` is a cudaStream_t passed as void*.  All work (kernels, NCCL) is
 *    enqueued on it; no call synchronises the host.  Host structs are read during
 *    the call and not retained.
 *  - Host-detectable errors (NULL pointers, bad sizes, k > 16, N > 32, workspace too
 *    small) return a non-OK status with NOTHING enqueued.  Data-dependent errors
 *    (token id >= V, parents[n] >= n or < -1, non-finite target logits) set bits in
 *    the device status word labels->status and the kernels still complete without
 *    undefined behaviour; the caller reads the word at its own sync point.
 *  - Row m = r*(N+1) + s: s = 0 is the root context (verifier logits after the
 *    prompt), s = n+1 the context after draft node n (the D_RPC l_t).
 *  - bf16 means IEEE bfloat16 bit patterns, row-major, densely packed unless an
 *    explicit leading dimension is given.
 *  - Nothing aborts; nothing prints.
 */
#ifndef AURORA_H_
#define AURORA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AURORA_ABI_VERSION 3
#define AURORA_MAX_NODES 32   /* N <= 32: one warp lane per draft node      */
#define AURORA_MAX_K 16       /* k_accept, k_discard <= 16 on the dense path */
#define AURORA_MAX_K_SPARSE 1024  /* k <= 1024 with the sparse top-K ingest (F1) */
#define AURORA_MAX_KT_SPARSE 16384 /* K_t limit when k > AURORA_MAX_K            */

typedef enum {
  AURORA_OK = 0,
  AURORA_ERR_INVALID_ARG = 1,   /* NULL pointer, bad size or stride              */
  AURORA_ERR_STRUCTURE = 2,     /* reserved: malformed parents (device word bit)  */
  AURORA_ERR_RANGE = 3,         /* reserved: token id >= V (device word bit)      */
  AURORA_ERR_NONFINITE = 4,     /* reserved: non-finite logits (device word bit)  */
  AURORA_ERR_UNSUPPORTED = 5,   /* valid request this build does not implement    */
  AURORA_ERR_WORKSPACE = 6,     /* ws NULL or ws_bytes < aurora_workspace_size()  */
  AURORA_ERR_CUDA = 7,          /* kernel launch / driver failure                 */
  AURORA_ERR_NCCL = 8           /* NCCL failure or NCCL unavailable               */
} aurora_status_t;

/* Bits of the device status word (labels->status[0]); OR-accumulated. */
#define AURORA_STATUS_NONFINITE 1u   /* a target logit is NaN or +-Inf           */
#define AURORA_STATUS_RANGE     2u   /* a draft token is < 0 or >= V             */
#define AURORA_STATUS_STRUCTURE 4u   /* parents[n] >= n or < -1                  */

/* Row classes (readings Q1-Q3 in DESIGN.md). */
#define AURORA_ROW_ACCEPT  0   /* root, or context of an accepted node       */
#define AURORA_ROW_DISCARD 1   /* context contains a rejected token  */
#define AURORA_ROW_PAD     2   /* ragged padding / out-of-scope discard: weight 0    */

/* Communicator for vocab-parallel (VP) / data-parallel (DP) runs.  NULL = 1 GPU. */
typedef struct aurora_comm_s* aurora_comm_t;

/* One local trace batch (P:372-376 D_RPC; S:397-410 TraceRecord). */
typedef struct {
  int32_t R;                     /* requests in this (local) batch, >= 1               */
  int32_t N;                     /* draft nodes per request, 1..32 (chain: gamma)      */
  const int32_t* draft_tokens;   /* (dev) int32 [R,N] proposed tokens, global vocab ids */
  const int32_t* parents;        /* (dev) int32 [R,N]; -1 = root, parents[n] < n
                                    (topological); NULL => chain, parent = n-1   */
  const int32_t* num_nodes;      /* (dev) int32 [R] valid nodes per request (ragged);
                                    NULL => all N.  Rows of nodes >= num_nodes are PAD. */
  const void* target_logits;     /* (dev) bf16 [M, ld_target] verifier logits over this
                                    rank's vocab slice [vocab_offset, vocab_offset+V_local) */
  int64_t ld_target;             /* row stride of target_logits in elements (>= V_local) */
  int64_t V;                     /* global vocabulary size                              */
  int64_t V_local;               /* vocab columns held by this rank                     */
  int64_t vocab_offset;          /* global id of local column 0                         */
} aurora_trace_t;

/* Loss configuration (Eq. 3; Table 3). */
typedef struct {
  int32_t k_accept;       /* support size on ACCEPT rows; default 1 = CE on the verified
                             token (reading Q5); 1..16 (dense verify), 1..1024
                             and <= K_t (sparse verify: soft distillation, F1)          */
  int32_t k_discard;      /* support size on DISCARD rows; default 10; same range.
                             0 = the paper's unfiltered "top-k 0": dense
                             KL(p_target || q) over the whole vocabulary (F2; dense
                             verify only; VP: the T row statistics are allgathered)     */
  float lambda_discard;   /* default 1.0; 0 disables the discard term          */
  int32_t normalize;      /* 0: per-term means over GLOBAL counts N_A, N_D (default,
                             S:378, reading Q7); 1: mean over N_A + N_D rows            */
  int32_t discard_scope;  /* 0: all rejected nodes (default); 1: only the first
                             rejected node on each branch (others become PAD)           */
  int32_t accept_loss;    /* ACCEPT-row objective (§5.1; NEXT F2):
                             0 = FKL KL(p~ || q) on the top-k_accept support (default);
                             1 = RKL KL(q || p_target) over the whole vocabulary,
                             gradient q*((ln q - ln p) - KL); dense verify only
                             (VP shards allgather per-row T statistics)                  */
  float ntp_beta;         /* >= 0: auxiliary NTP cross-entropy -ln q_y on ACCEPT rows,
                             y = verified token, weight beta x the row weight ("RKL +
                             NTP"); requires accept_loss = 1           */
  int32_t discard_restricted; /* 0 (default): DISCARD rows use the full-vocabulary log-softmax
                             (reading Q6); 1: SPEC's restricted softmax: both
                             distributions renormalised over the top-k_discard support,
                             KL(p~ || q~) with q~ = softmax of the support logits, gradient
                             q~ - p~ on the support and zero elsewhere (NEXT F2).  Requires
                             accept_loss = 0, k_discard >= 1, the staged forward (ws of
                             AURORA_OP_ALL, one dZ^T chunk) and no VP group; the row's support
                             log-sum-exp is written to labels->row_aux                       */
} aurora_loss_cfg_t;

/* Caller-allocated outputs of verify; inputs of fwd/bwd.  All (dev). */
typedef struct {
  int32_t k_max;          /* (in) row stride of sup_idx/sup_p; >= max(k_accept,k_discard);
                             <= 16 for aurora_verify_labels, <= 1024 otherwise           */
  int32_t* target_argmax; /* [M]  y_m, global id; lowest index wins ties  */
  uint8_t* accepted;      /* [R,N] 1 = node on the accepted path                         */
  int32_t* accept_len;    /* [R]  #accepted + 1 (bonus counts)                    */
  int32_t* bonus;         /* [R]  y at the deepest accepted row                          */
  uint8_t* row_class;     /* [M]  AURORA_ROW_*                                           */
  int32_t* sup_idx;       /* [M,k_max] target top-k support, GLOBAL ids sorted ascending;
                             unused slots = INT32_MAX                                    */
  float* sup_p;           /* [M,k_max] renormalised target probs p~ aligned with sup_idx */
  float* row_H;           /* [M]  sum_j p~ log p~ (0 when k = 1)                          */
  float* row_w;           /* [M]  loss weight: 1/N_A, lambda/N_D or 0                     */
  int32_t* counts;        /* [2]  N_A, N_D (global over DP ranks)                        */
  uint32_t* status;       /* [1]  device status word, AURORA_STATUS_* bits                */
  /* NEXT F2 (accept_loss = 1 or k_discard = 0; otherwise may be NULL / 0):            */
  float* row_lse_t;          /* [M] written by verify: log sum_j exp(T_mj), full row      */
  float* row_aux;            /* [M] written by fwd, read by bwd: E_q[z - t] on RKL rows   */
  const void* target_logits; /* (in) the bf16 T given to verify ([M, ld_target], this
                                rank's vocab slice); fwd and bwd read its tiles again, so it
                                must stay valid until the bwd call has run                 */
  int64_t ld_target;         /* row stride of target_logits in elements                     */
  int32_t objective;         /* written by verify: bit 0 RKL ACCEPT rows, bit 1 dense-KL
                                DISCARD rows, bit 2 restricted-softmax DISCARD rows (0 = Eq. 3
                                everywhere); read by fwd / bwd                              */
  float ntp_beta;            /* written by verify: cfg->ntp_beta                             */
} aurora_labels_t;

/* Workspace sizing.  op: 0 = verify, 1 = fwd, 2 = bwd, 3 = max over all three.
 * Depends only on the arguments; a buffer of the returned size (256-byte aligned
 * base) may be reused for every call with the same sizes.  Returns 0 on bad args. */
#define AURORA_OP_VERIFY 0
#define AURORA_OP_FWD 1
#define AURORA_OP_BWD 2
#define AURORA_OP_ALL 3
size_t aurora_workspace_size(int op, int64_t M, int64_t d, int64_t V_local,
                             const aurora_loss_cfg_t* cfg);

/* Greedy verification + labels.
 * Scans every target row once (argmax + top-k_max, exact bf16 compares), verifies
 * chains/trees (acc(n) = acc(parent) AND x_n == y_row(parent); lowest-index sibling
 * wins, reading Q12), classifies rows, builds supports p~ and weights w.
 * VP: candidates are merged across ranks (global order), DP: counts are summed. */
aurora_status_t aurora_verify_labels(const aurora_trace_t* trace, const aurora_loss_cfg_t* cfg,
                                     aurora_labels_t* out, void* ws, size_t ws_bytes,
                                     aurora_comm_t comm, void* stream);

/* NEXT F1 — sparse target ingest: the verifier's logits arrive as the paper's transmitted
 * top-K payload ("top-K logits filtering (e.g., K=1024)").
 * Same verification and targets as aurora_verify_labels, computed from the pairs. */
typedef struct {
  int32_t R, N;                  /* as aurora_trace_t                                      */
  const int32_t* draft_tokens;   /* (dev) int32 [R,N]                                      */
  const int32_t* parents;        /* (dev) int32 [R,N] or NULL (chain)                      */
  const int32_t* num_nodes;      /* (dev) int32 [R] or NULL                                */
  const int32_t* target_ids;     /* (dev) int32 [M, K_t] global vocab ids, distinct per row,
                                    any order                                              */
  const void* target_vals;       /* (dev) bf16 [M, K_t] verifier logits of those ids       */
  int32_t K_t;                   /* transmitted pairs per row, >= max(k_accept, k_discard) */
  int64_t V;                     /* global vocabulary size                                 */
} aurora_trace_topk_t;

/* argmax / top-k are taken over the K_t transmitted pairs by (value desc, id asc);
 * status bits: non-finite logit, id outside [0, V) (pair skipped), an id seen twice in the
 * top list (STRUCTURE).  Workspace: aurora_workspace_size(AURORA_OP_VERIFY, M, d, K_t, cfg).
 * k = max(k_accept, k_discard) <= 16: warp-list scan; 16 < k <= 1024 (soft distillation
 * over up to the whole payload): CTA-per-row bitonic sort, K_t <= 16384.
 * VP ranks each hold the full payload (no candidate exchange); DP sums the counts. */
aurora_status_t aurora_verify_labels_topk(const aurora_trace_topk_t* trace, const aurora_loss_cfg_t* cfg,
                                          aurora_labels_t* out, void* ws, size_t ws_bytes,
                                          aurora_comm_t comm, void* stream);

/* Forward (Eq. 3).
 * H (dev) bf16 [M,d] draft-head hidden states; W (dev) bf16 [V_local,d] lm_head rows
 * for global ids [vocab_offset, vocab_offset+V_local).  d % 64 == 0.
 * Outputs: row_lse (dev) f32 [M] = log sum_j exp(z_mj) over the GLOBAL vocabulary;
 * row_loss (dev, nullable) f32 [M] = KL(p~_m || softmax(z_m)); loss (dev) f32 [1] =
 * sum_m w_m row_loss_m.  Z = H W^T is consumed tile by tile in TMEM. */
aurora_status_t aurora_spec_loss_fwd(const void* H, const void* W, int64_t M, int64_t d,
                                     int64_t V_local, int64_t vocab_offset,
                                     const aurora_labels_t* labels, float* row_lse,
                                     float* row_loss, float* loss, void* ws, size_t ws_bytes,
                                     aurora_comm_t comm, void* stream);

/* Backward.  dz_mj = g w_m (exp(z_mj - lse_m) - p~_mj) is
 * recomputed per tile, rounded to bf16 into a per-vocab-chunk workspace, then
 * dW[chunk] = dZ^T H and dH += dZ W[chunk].
 * dloss (dev, nullable => g = 1) f32 [1] upstream gradient.
 * dH (dev) f32 [M,d] (overwritten; VP: summed over ranks).
 * dW (dev) [V_local,d]: f32 (dW_is_bf16 = 0, P:495 fp32 gradients) or bf16 (dW_is_bf16 = 1:
 * the GEMM's fp32 accumulators rounded once; not with accumulation, an unreduced DP group or
 * the fused persistent backward -> UNSUPPORTED).  accumulate_dW: bit 0 (AURORA_BWD_ACCUMULATE) adds into dW (micro-batch
 * accumulation); bit 1 (AURORA_BWD_NO_DP_REDUCE) skips the DP dW allreduce (C5)
 * because the caller reduce-scatters it in aurora_adamw_step_sharded. */
#define AURORA_BWD_ACCUMULATE 1
#define AURORA_BWD_NO_DP_REDUCE 2
aurora_status_t aurora_spec_loss_bwd(const void* H, const void* W, int64_t M, int64_t d,
                                     int64_t V_local, int64_t vocab_offset,
                                     const aurora_labels_t* labels, const float* row_lse,
                                     const float* dloss, float* dH, void* dW, int dW_is_bf16,
                                     int accumulate_dW, void* ws, size_t ws_bytes,
                                     aurora_comm_t comm, void* stream);

/* Communicator (vocab-parallel x data-parallel, one process per GPU).
 * nccl_unique_id (host) points to the 128-byte ncclUniqueId that rank 0 created with
 * aurora_comm_get_unique_id and the caller broadcast (e.g. torch.distributed).
 * Ranks are laid out dp-major: rank = dp_rank * vp_size + vp_rank.  A group exchanges
 * (C1-C5) iff its size > 1; a communicator with nranks == 1 runs every exchange as an
 * identity collective (used to test the NCCL plumbing on one GPU).  The comm owns a
 * small device scratch for gathered per-row data that grows on first use. */
aurora_status_t aurora_comm_get_unique_id(void* nccl_unique_id_out /* 128 bytes */);
aurora_status_t aurora_comm_create(const void* nccl_unique_id, int nranks, int rank,
                                   int vp_size, int dp_size, aurora_comm_t* out);
aurora_status_t aurora_comm_destroy(aurora_comm_t comm);
/* Loopback communicator: `nranks` = vp_size x dp_size VIRTUAL ranks on the current device
 * (same rank layout as above), written to out[0 .. nranks-1] (host array, caller-owned;
 * each handle released with aurora_comm_destroy).  Each virtual rank must be driven from
 * its own host thread on its own stream, issuing the same calls in the same order as a
 * real rank would (SPMD); the collectives are device copies into a group-shared staging
 * buffer, ordered by CUDA events plus a host barrier per collective, and the sums run in
 * rank order (deterministic).  Not capturable into a CUDA graph.  Purpose: execute the
 * library's multi-rank code (C1-C5, the F2 merge, the DP reduce-scatter) on one GPU and
 * check it against the single-process oracle. */
aurora_status_t aurora_comm_create_loopback(int nranks, int vp_size, int dp_size, aurora_comm_t* out);

const char* aurora_status_string(aurora_status_t s);
/* Static build information ("sm_100a, tcgen05 ..."). */
const char* aurora_build_info(void);
/* Number of kernels this library has launched since load (for bench accounting). */
uint64_t aurora_launch_count(void);

/* Execution options (process-wide; affect performance only, never results beyond fp32
 * summation order).  Defaults come from the environment (AURORA_PAIR, AURORA_BWD,
 * AURORA_SERIAL_BWD).  Returns AURORA_ERR_INVALID_ARG for an unknown name or value.
 *   "gemm_pair"      0 auto (default), 1 single-CTA 128x256 tiles, 2 CTA-pair 256x256
 *                    tiles (tcgen05.mma.cta_group::2)
 *   "bwd_mode"       0 per-chunk launches (default), 1 one fused persistent kernel
 *   "bwd_concurrent" 0 (default): serial; 1: dW || dH of a chunk on library side streams
 *   "dw_resident"    0 (default): streamed pair tiles for dW; 1: with K = M <= 512 each CTA
 *                    pair keeps its dZ^T rows in shared memory across all column tiles
 *   "scan_ctas"      target-scan CTAs per SM (row segments) of the (row, segment) scan, default 2
 *   "scan_flat"      1 (default): load-balanced scan (the batch's 16 B vectors cut into equal
 *                    contiguous ranges per warp; rows 16 B aligned, V_local % 8 == 0) where the
 *                    (row, segment) grid would leave a wave tail (>= 2 waves, last one under
 *                    half full), else the (row, segment) scan; 2: always the load-balanced
 *                    scan (when aligned); 0: always the (row, segment) scan
 *   "dz_chunk_bytes" budget of the bwd's bf16 dZ^T chunk (default 16 GiB: the whole local
 *                    vocabulary at the bench shapes; smaller -> more chunks).  Options that
 *                    change workspace sizes must be set before aurora_workspace_size.
 *   "tile_n"         fwd / dz vocab tile width with single-CTA tiles: 0 auto (default:
 *                    the width among 256/224/192 with the least per-SM work for the
 *                    tile count), or force 256, 224 or 192.
 *   "tree_fwd_tc"    tree-attention forward when (Hq/Hkv)*(N+1) <= 128: 2 (default) one-pass
 *                    tcgen05 kernel, two work items per SM; 3 the same with one item and deeper
 *                    K/V rings; 1 two-pass tcgen05 kernel; 0 the mma.sync kernel
 *   "tree_bwd_tc"    tree-attention backward when (Hq/Hkv)*(N+1) <= 128: 1 (default) tcgen05
 *                    one-kernel backward; 0 the mma.sync one-kernel backward
 *   "tree_bwd_split" 1: the general dQ + dK/dV mma.sync kernels even where the one-kernel
 *                    backward applies (always used when (Hq/Hkv)*(N+1) > 128)
 *   Other values: INVALID_ARG. */
aurora_status_t aurora_set_option(const char* name, int64_t value);
int64_t aurora_get_option(const char* name);

/* NEXT F3 — the optimizer step on the (vocab-sharded) lm_head, Table 3 P:507-515:
 * AdamW (decoupled weight decay, default 0.0), global-norm gradient clipping (max norm
 * 0.5), linear warm-up over warmup_steps then a constant learning rate (S:379:
 * lr(s) = lr * s / warmup for s < warmup).  "FP32 master weights and gradients cast to
 * FP32 before optimization": W_master, m, v, dW are fp32; the bf16 copy the
 * GEMMs read is rewritten from the updated master.
 *   W_master, m, v (dev) f32 [n], updated in place; W_bf16 (dev, nullable) bf16 [n] out;
 *   dW (dev) f32 [n]; step >= 1: the step number (bias corrections 1 - beta^step, warm-up);
 *   step = 0: the step counter kept on the device in `ws` (an int64 the call increments
 *   before using it; a zero-filled workspace starts at step 1), so a CUDA graph that
 *   captured the call advances the schedule on every replay;
 *   extra_sq (dev, nullable) f32 [1]: sum of squares of the gradients of parameters
 *   outside this call (they share the global norm; added once, AFTER the VP allreduce,
 *   so it must hold the sum over every rank's other groups, e.g. replicated parameters
 *   counted once); grad_norm (dev, nullable) f32 [1] out: the global norm before
 *   clipping.  comm: norm^2 of dW is summed over the VP group (disjoint vocab shards); DP
 *   replicas hold the already-reduced dW (C5) — or use aurora_adamw_step_sharded.
 *   n % 4 == 0 and 16-byte aligned pointers.  Deterministic (fixed reduction order). */
typedef struct {
  float lr;              /* base learning rate (1e-5 finetune / 1e-4 scratch)  */
  float beta1, beta2;    /* 0.9, 0.999 (SPEC design decision; paper silent)            */
  float eps;             /* 1e-8                                                        */
  float weight_decay;    /* 0.0 (Table 3)                                               */
  float max_grad_norm;   /* 0.5 (Table 3); <= 0 disables clipping                        */
  int32_t warmup_steps;  /* 400; 0 = constant from step 1                       */
} aurora_adamw_cfg_t;
size_t aurora_adamw_workspace_size(int64_t n);
aurora_status_t aurora_adamw_step(float* W_master, void* W_bf16, float* m, float* v, const float* dW, int64_t n,
                                  int64_t step, const aurora_adamw_cfg_t* cfg, const float* extra_sq,
                                  float* grad_norm, void* ws, size_t ws_bytes, aurora_comm_t comm, void* stream);

/* F3 under data parallelism (ZeRO-style sharded optimizer state; P:487-489 optimizer,
 * P:495 fp32 master and gradients).  dW (dev f32 [n]): this rank's UNREDUCED gradient of
 * its (VP-local) lm_head, from aurora_spec_loss_bwd with AURORA_BWD_NO_DP_REDUCE.  It is
 * reduce-scattered over the DP group (replacing the C5 allreduce: half the traffic); DP
 * rank q owns elements [q n/P, (q+1) n/P) of the optimizer state: W_master_shard, m_shard,
 * v_shard (dev f32 [n/P], updated in place).  The global norm sums the shards over the DP
 * and VP groups (+ extra_sq once); after the update the bf16 shards are allgathered into
 * W_bf16 (dev bf16 [n], every rank's full copy the GEMMs read).  comm required (a 1-rank
 * or DP-1 comm degenerates to aurora_adamw_step); n % (4 P) == 0; 16-byte aligned
 * pointers; step as in aurora_adamw_step (0 = device counter in ws).  ws:
 * aurora_adamw_sharded_workspace_size(n, P) bytes. */
size_t aurora_adamw_sharded_workspace_size(int64_t n, int dp_size);
aurora_status_t aurora_adamw_step_sharded(float* W_master_shard, void* W_bf16, float* m_shard, float* v_shard,
                                          const float* dW, int64_t n, int64_t step,
                                          const aurora_adamw_cfg_t* cfg, const float* extra_sq,
                                          float* grad_norm, void* ws, size_t ws_bytes,
                                          aurora_comm_t comm, void* stream);

/* NEXT F3, fused with the backward (SURVEY F3 "applied from the dW epilogue"): runs the
 * backward of aurora_spec_loss_bwd for dH, then the optimizer step of aurora_adamw_step on
 * the fp32 master lm_head WITHOUT materialising dW: the dW GEMM is recomputed from the
 * bf16 dZ^T the backward left in `ws`, once for the global gradient norm (sum of squares
 * in the epilogue) and once with the AdamW update applied from the TMEM accumulators
 * (m, v and the fp32 master streamed through shared memory by TMA; 26 B per element).  W (bf16 [V_local, d])
 * is rewritten from the updated master after dz and dH have read it.  Requires the whole
 * local vocabulary in one dZ^T chunk (option dz_chunk_bytes) and a DP group of size 1 (the DP dW
 * allreduce must precede the optimizer: use aurora_spec_loss_bwd + aurora_adamw_step);
 * otherwise UNSUPPORTED.  opt_ws: aurora_adamw_workspace_size(V_local * d) bytes. */
aurora_status_t aurora_spec_loss_bwd_adamw(const void* H, void* W, int64_t M, int64_t d, int64_t V_local,
                                           int64_t vocab_offset, const aurora_labels_t* labels,
                                           const float* row_lse, const float* dloss, float* dH,
                                           float* W_master, float* m, float* v, int64_t step,
                                           const aurora_adamw_cfg_t* cfg, const float* extra_sq,
                                           float* grad_norm, void* ws, size_t ws_bytes, void* opt_ws,
                                           size_t opt_ws_bytes, aurora_comm_t comm, void* stream);

/* ---- NEXT F4: tree attention of the draft layer -------------------------------------
 * P:163-169 §3.2 "Efficient Tree Attention ... a custom attention mask that respects the
 * causal structure of the speculative tree ... all accepted and rejected branches in a
 * single batched forward and backward pass"; the tree is S:134-140 (parents[n] < n).
 * Readings F4-R1..R5:
 *  - request r has P_r prefix positions (K/V given: the draft layer's cached prefix, packed
 *    [P_total, Hkv, dh], request r at rows prefix_off[r] .. prefix_off[r+1]-1) and N+1 tree
 *    rows in the lm_head path's order (s = 0 root, s = n+1 draft node n);
 *  - tree row s attends every prefix position of its request and the tree rows in its
 *    ancestor closure anc*(s) (its ancestors, the root and itself) — never a sibling
 *    branch; rows of padded nodes (n >= num_nodes[r]) are keys of nobody and, as queries,
 *    produce O = 0, lse = -inf and zero gradients;
 *  - GQA: query head h reads kv head h / (Hq / Hkv).
 *  O = softmax(scale * Q K^T + mask) V per (row, head); lse = natural log-sum-exp of the
 *  scaled, masked scores.  Backward: the gradients of <dO, O> (textbook softmax-attention
 *  backward), with dK/dV of a kv head summed over its Hq/Hkv query heads.
 * Layouts (bf16 unless stated, dense row-major):
 *  Q, O, dO [R, N+1, Hq, dh]; Kt, Vt, dKt, dVt [R, N+1, Hkv, dh]; Kp, Vp, dKp, dVp
 *  [P_total, Hkv, dh]; lse f32 [R, N+1, Hq]; dQ f32 [R, N+1, Hq, dh].
 * Limits (else UNSUPPORTED, nothing enqueued): dh == 128, 1 <= N <= 32, Hq % Hkv == 0,
 * (Hq/Hkv)*(N+1) <= 256, R <= 65535.  NULL or non-16-byte-aligned tensors: INVALID_ARG; a
 * backward workspace below aurora_tree_attn_workspace_size(): WORKSPACE.  Data errors OR bits into *status (if non-NULL): STRUCTURE for a
 * malformed parent array or num_nodes outside [0, N] (that request's rows are treated as
 * padding), RANGE for a prefix longer than max_prefix (its keys beyond max_prefix are
 * ignored). */
typedef struct {
  int32_t R, N, Hq, Hkv, dh;
  int32_t max_prefix;            /* host bound on every P_r (sizes the backward grid)    */
  int64_t prefix_total;          /* rows of Kp / Vp (= prefix_off[R]; bounds the TMA maps) */
  const int32_t* prefix_off;     /* (dev) int32 [R+1], prefix_off[0] = 0, non-decreasing  */
  const int32_t* parents;        /* (dev) int32 [R,N] or NULL (chain)                    */
  const int32_t* num_nodes;      /* (dev) int32 [R] or NULL (all N)                      */
  float scale;                   /* softmax scale; <= 0 means 1/sqrt(dh)                 */
  uint32_t* status;              /* (dev) optional OR-accumulated status word            */
} aurora_tree_attn_t;

aurora_status_t aurora_tree_attn_fwd(const aurora_tree_attn_t* ta, const void* Q, const void* Kt,
                                     const void* Vt, const void* Kp, const void* Vp, void* O, float* lse,
                                     void* stream);
/* Scratch of the backward: 4 B per (row, query head) (the rowsum(dO * O) terms). */
size_t aurora_tree_attn_workspace_size(const aurora_tree_attn_t* ta);
/* dKp/dVp/dKt/dVt are overwritten (every element: keys nobody attends get 0). */
aurora_status_t aurora_tree_attn_bwd(const aurora_tree_attn_t* ta, const void* Q, const void* Kt,
                                     const void* Vt, const void* Kp, const void* Vp, const void* O,
                                     const float* lse, const void* dO, float* dQ, void* dKt, void* dVt,
                                     void* dKp, void* dVp, void* ws, size_t ws_bytes, void* stream);

/* Tree positions + RoPE (F4-R6): tree row s of request r sits at position P_r + depth(s)
 * (root depth 0; siblings share a position); rotates, in place, Q [R, N+1, Hq, dh] and the tree
 * keys Kt [R, N+1, Hkv, dh] there with the rotate-half convention (pairs (i, i + dh/2), angle
 * pos * theta^(-2i/dh)); inverse != 0 applies the transposed rotation (dQ / dKt of the rotated
 * tensors -> gradients of the unrotated ones).  Q or Kt may be NULL (skipped); *_fp32 selects
 * f32 instead of bf16 storage.  Padded / malformed rows are left unrotated (STRUCTURE bit for
 * malformed parents, as the attention kernels).  The cached prefix keys are not touched (already
 * rotated at positions 0..P_r-1).  Limits: dh even, <= 256; theta > 1. */
aurora_status_t aurora_tree_rope(const aurora_tree_attn_t* ta, void* Q, int q_fp32, void* Kt, int kt_fp32,
                                 float theta, int inverse, void* stream);

/* ---- NEXT F4: the EAGLE-3 draft layer around the tree attention (reading F4-R7) ----------
 *   g = h3 Wfc^T;  u = [rms(e) w_e ; rms(g) w_h];  q,k,v = u W{q,k,v}^T;  RoPE(q, k) at tree
 *   positions (aurora_tree_rope);  o = tree attention over [Kp; k], [Vp; v];  y = g + o Wo^T;
 *   z = rms(y) w_post;  h = y + (silu(z Wg^T) * (z Wu^T)) Wd^T;  H = rms(h) w_final (the final
 *   norm before the lm_head),   rms(x) = x (mean x^2 + eps)^-1/2
 * Rows in the lm_head path's order, M = R (N+1).  Layouts (row-major, dense): h3 bf16 [M, 3d],
 * e bf16 [M, d] (token embeddings), H bf16 [M, d]; Wfc [d, 3d], Wq [Hq dh, 2d], Wk/Wv [Hkv dh, 2d],
 * Wo [d, Hq dh], Wg/Wu [I, d], Wd [d, I] bf16 (nn.Linear); w_e, w_h, w_post, w_final f32 [d].  The
 * dense projections run on the library's tcgen05 GEMM engine (bf16 operands, fp32 accumulation in
 * TMEM, bf16 / fp32 TMA-store epilogues, residual adds as TMA reduce-add).  aurora_draft_layer_fwd
 * keeps the activations the backward needs in `ws` (aurora_draft_layer_workspace_size bytes); the
 * matching aurora_draft_layer_bwd must get the same ws.  Gradients: weights f32 (overwritten),
 * dh3 / de f32 [M, 3d] / [M, d], dKp / dVp bf16 like Kp / Vp.  Limits: dh == 128 (tree attention),
 * d and I multiples of 64, eps > 0; else UNSUPPORTED / INVALID_ARG with nothing enqueued. */
typedef struct {
  aurora_tree_attn_t ta;         /* batch structure, heads (Hq, Hkv, dh), prefix bounds, status */
  int32_t d, I;                  /* hidden size, MLP intermediate size                          */
  float theta, eps;              /* RoPE base, RMSNorm epsilon                                  */
} aurora_draft_layer_t;
typedef struct {
  const void *Wfc, *Wq, *Wk, *Wv, *Wo, *Wg, *Wu, *Wd;   /* (dev) bf16 */
  const float *we, *wh, *wpost, *wfinal;                 /* (dev) f32  */
} aurora_draft_weights_t;
typedef struct {
  float *Wfc, *Wq, *Wk, *Wv, *Wo, *Wg, *Wu, *Wd, *we, *wh, *wpost, *wfinal;  /* (dev) f32, overwritten */
} aurora_draft_grads_t;
size_t aurora_draft_layer_workspace_size(const aurora_draft_layer_t* L);
aurora_status_t aurora_draft_layer_fwd(const aurora_draft_layer_t* L, const aurora_draft_weights_t* W, const void* h3,
                                       const void* e, const void* Kp, const void* Vp, void* H, void* ws,
                                       size_t ws_bytes, void* stream);
aurora_status_t aurora_draft_layer_bwd(const aurora_draft_layer_t* L, const aurora_draft_weights_t* W, const void* h3,
                                       const void* e, const void* Kp, const void* Vp, const float* dH,
                                       const aurora_draft_grads_t* G, float* dh3, float* de, void* dKp, void* dVp,
                                       void* ws, size_t ws_bytes, void* stream);

/* Per-phase device timing (CUDA events recorded on the caller's stream around each
 * phase while enabled).  aurora_profile_read must be called after the stream was
 * synchronised; it fills up to `max` (name, total ms, launches) triples and returns
 * the number of phases, then clears the accumulators. */
void aurora_profile_enable(int enable);
int aurora_profile_read(const char** names, float* total_ms, int32_t* count, int max);
/* As aurora_profile_read but keeps the recorded events: phases captured into a CUDA graph
 * (recorded there as external event nodes) are re-timed by every replay; peek after each
 * replay returns that replay's per-phase times. */
int aurora_profile_peek(const char** names, float* total_ms, int32_t* count, int max);

/* ---- Test hooks (not on the hot path) ------------------------------------ */
/* D[M,N] (dev f32, ld ldd) = sum_k A(m,k) B(n,k) on the tcgen05 GEMM engine.
 * a_mn_major = 0: A is bf16 [M,K] (ld lda); 1: A is stored as bf16 [K,M] (ld lda).
 * b_mn_major = 0: B is bf16 [N,K] (ld ldb); 1: B is stored as bf16 [K,N] (ld ldb). */
aurora_status_t aurora_debug_gemm(int a_mn_major, int b_mn_major, const void* A, const void* B,
                                  float* D, int64_t M, int64_t N, int64_t K, int64_t lda,
                                  int64_t ldb, int64_t ldd, void* stream);
/* out (dev f32 [n_rows, V_local]) = full dLogits rows dz for the listed rows (dev int32). */
aurora_status_t aurora_debug_dlogits_rows(const void* H, const void* W, int64_t M, int64_t d,
                                          int64_t V_local, int64_t vocab_offset,
                                          const aurora_labels_t* labels, const float* row_lse,
                                          const float* dloss, const int32_t* rows, int32_t n_rows,
                                          float* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* AURORA_H_ */

"""Seeded synthetic trace generator — shared by tests, bench.py and smoke().

This module only *draws* inputs. It holds none of the method's arithmetic: it
never computes an argmax, a verification outcome, a support set, a softmax or a
loss. Those live in `oracle/` (CPU checker) and in the CUDA library (product),
which share no code. Both consume the same raw bit patterns produced here.

A trace batch is the per-step input contract of the hot path (
PAPER.md:372-376, App. A, the D_RPC payload (h_t, l_t, x_in, y_out, R)):

  draft_tokens  int32 [R, N]       the draft's proposed tokens per node
  parents       int32 [R, N]       -1 = root, parents[n] < n; None => chain
  num_nodes     int32 [R]          ragged valid-node count; None => N
  T_bits        uint16 [M, V]      bf16 bit patterns of the verifier logits,
                                   row m = r*(N+1) + s (s=0 root, s=n+1 after node n)
  H_bits        uint16 [M, d]      bf16 draft-head hidden states (same row order)
  W_bits        uint16 [V, d]      bf16 lm_head weight (nn.Linear layout, no bias)

Recipe (restated in DESIGN.md "Input recipe"):
  * numpy Generator(PCG64(seed)); draws in a fixed order W, H, tokens, parents,
    alpha, T.
  * H ~ N(0,1), W ~ N(0, (2/sqrt(d))^2), both rounded to bf16 (RNE), so a
    logit z = h.w has std ~2.
  * draft tokens follow Zipf(1.1) over a seeded vocab permutation; siblings
    are distinct.
  * T rows ~ N(0, 2^2); the row's *designated* next token gets row max + 1.0
    (before bf16 rounding) so it is the strict maximum; natural bf16 ties among
    the rest of the top-10 are kept.  With probability alpha the designated
    token of a row equals the token of (one of) the node(s) whose parent is
    that row — that is how an acceptance rate is planted.  Whether a node is
    accepted is decided later by the oracle / kernels from the bits, not here.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

__all__ = ["TraceConfig", "CONFIGS", "gen_trace", "gen_trace_topk", "f32_to_bf16_bits", "bf16_bits_to_f32",
           "TreeAttnConfig", "TREE_ATTN_CONFIGS", "gen_tree_attn", "gen_tree_attn_meta"]


@dataclasses.dataclass(frozen=True)
class TraceConfig:
    name: str
    d: int
    V: int
    R: int
    N: int                      # nodes per request (chain: gamma)
    seed: int
    tree: bool = False          # beam tree (width `beam`) instead of a chain
    beam: int = 4
    alpha: tuple = (0.79,)      # per-request-block acceptance probabilities
    ragged: bool = False        # draw num_nodes < N for some requests
    inject_ties: bool = False   # tiny config: exact ties at argmax / k-th place, +-0

    @property
    def M(self) -> int:
        return self.R * (self.N + 1)


# BASELINE.json "configs" (index order kept) plus small parity-only shapes.
CONFIGS = {
    # configs[0]: "tiny oracle case: hidden=64, vocab=1000, 4 requests x draft depth 4 (chain)"
    "tiny": TraceConfig("tiny", d=64, V=1000, R=4, N=4, seed=1001, alpha=(0.6,), inject_ties=True),
    # configs[1]: Llama-3.1-8B speculator, alpha 0.79 => E[L]=3.60 ("~3.6 at lookahead 5")
    "llama": TraceConfig("llama", d=4096, V=128256, R=64, N=5, seed=1002, alpha=(0.79,)),
    # configs[2]: Qwen3-8B, ordered two-domain stream: alpha 0.75 then 0.35
    "qwen3": TraceConfig("qwen3", d=4096, V=151936, R=256, N=6, seed=1003, alpha=(0.75, 0.35)),
    # configs[3]: MiniMax-M2.1-shaped, alpha 0.65 => E[L]=2.80 ("2.8")
    "minimax": TraceConfig("minimax", d=3072, V=200064, R=512, N=8, seed=1004, alpha=(0.65,)),
    # configs[4]: tree drafts, beam 4 x depth 6 = 24 nodes, Qwen3 vocab
    "tree": TraceConfig("tree", d=4096, V=151936, R=1024, N=24, seed=1005, tree=True, beam=4, alpha=(0.7,)),
    # NEXT F1 shipping format: the Llama-3 draft's 32K draft vocabulary ("32K vs
    # 128K for Llama3"); used with gen_trace_topk (top-1024 pairs over the draft vocab)
    "llama_d32k": TraceConfig("llama_d32k", d=4096, V=32000, R=64, N=5, seed=1006, alpha=(0.79,)),
    # parity-only shapes: several tiles plus ragged vocab/row tails, oracle finishes in seconds
    "small": TraceConfig("small", d=256, V=5003, R=13, N=5, seed=2001, alpha=(0.7,), ragged=True),
    "small_tree": TraceConfig("small_tree", d=192, V=3001, R=9, N=12, seed=2002, tree=True, beam=3, alpha=(0.7,)),
    "mid": TraceConfig("mid", d=1024, V=20000, R=40, N=6, seed=2003, alpha=(0.75, 0.35)),
}


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round float32 -> bf16 (round to nearest even), returned as uint16 bits."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def _zipf_tokens(rng: np.random.Generator, perm: np.ndarray, size: int, V: int) -> np.ndarray:
    # Zipf(1.1) ranks, folded into [0, V), mapped through a seeded permutation so
    # frequent ids scatter across vocab tiles.
    ranks = rng.zipf(1.1, size=size) - 1
    ranks = ranks % V
    return perm[ranks]


def _distinct_from(rng, perm, V, forbid: set) -> int:
    while True:
        t = int(_zipf_tokens(rng, perm, 1, V)[0])
        if t not in forbid:
            return t


def _tree_parents(rng: np.random.Generator, R: int, depth: int, beam: int) -> np.ndarray:
    """Beam tree: level 1 = `beam` children of the root; level l = `beam` nodes whose
    parents are drawn from level l-1 with rank weights (0.55, 0.25, 0.12, 0.08)."""
    w = np.array([0.55, 0.25, 0.12, 0.08][:beam], dtype=np.float64)
    if beam > 4:
        w = np.concatenate([w, np.full(beam - 4, 0.02)])
    w = w / w.sum()
    N = depth * beam
    parents = np.empty((R, N), dtype=np.int32)
    for r in range(R):
        parents[r, :beam] = -1
        for lvl in range(1, depth):
            prev0 = (lvl - 1) * beam
            picks = rng.choice(beam, size=beam, p=w)
            picks.sort()                       # keep children of a parent contiguous
            parents[r, lvl * beam:(lvl + 1) * beam] = prev0 + picks
    return parents


def gen_trace(cfg: TraceConfig | str, seed: Optional[int] = None, rows: Optional[np.ndarray] = None,
              gen_T: bool = True, gen_W: bool = True) -> dict:
    """Generate one trace batch. `rows` is unused (kept for API symmetry).  gen_W=False
    skips the W draw (bench.py's multi-GPU legs draw W and T slices on the device); the
    later draws then come from a different position of the stream."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    seed = cfg.seed if seed is None else seed
    rng = np.random.Generator(np.random.PCG64(seed))
    d, V, R, N = cfg.d, cfg.V, cfg.R, cfg.N
    M = R * (N + 1)

    # --- W, H (bf16) -------------------------------------------------------
    W_bits = np.empty((V, d) if gen_W else (0, d), dtype=np.uint16)
    step = max(1, (1 << 24) // d)
    for v0 in range(0, V if gen_W else 0, step):
        v1 = min(V, v0 + step)
        W_bits[v0:v1] = f32_to_bf16_bits(rng.standard_normal((v1 - v0, d), dtype=np.float32)
                                         * np.float32(2.0 / math.sqrt(d)))
    H_bits = f32_to_bf16_bits(rng.standard_normal((M, d), dtype=np.float32))

    # --- draft tokens / parents -------------------------------------------
    perm = rng.permutation(V).astype(np.int64)
    if cfg.tree:
        depth = N // cfg.beam
        assert depth * cfg.beam == N
        parents = _tree_parents(rng, R, depth, cfg.beam)
    else:
        parents = None
    draft = np.empty((R, N), dtype=np.int32)
    for r in range(R):
        if parents is None:
            draft[r] = _zipf_tokens(rng, perm, N, V)
        else:
            for n in range(N):
                sib = {int(draft[r, s]) for s in range(n) if parents[r, s] == parents[r, n]}
                draft[r, n] = _distinct_from(rng, perm, V, sib)
    num_nodes = None
    if cfg.ragged:
        num_nodes = np.full(R, N, dtype=np.int32)
        for r in range(R):
            if rng.random() < 0.4:
                num_nodes[r] = int(rng.integers(0, N))       # 0..N-1 valid nodes

    # --- alpha per request (ordered stream blocks) -------------------------
    nblk = len(cfg.alpha)
    alpha_r = np.array([cfg.alpha[min(nblk - 1, r * nblk // R)] for r in range(R)])

    # --- designated next token per row -------------------------------------
    # children of row s: chain -> node s (if s < N); tree -> nodes with parent s-1
    designated = np.empty(M, dtype=np.int64)
    for r in range(R):
        nn = N if num_nodes is None else int(num_nodes[r])
        for s in range(N + 1):
            m = r * (N + 1) + s
            if parents is None:
                kids = [s] if s < nn else []
            else:
                kids = [n for n in range(nn) if parents[r, n] == s - 1]
            kid_tokens = [int(draft[r, n]) for n in kids]
            if kid_tokens and rng.random() < alpha_r[r]:
                designated[m] = kid_tokens[int(rng.integers(0, len(kid_tokens)))]
            else:
                designated[m] = _distinct_from(rng, perm, V, set(kid_tokens))

    out = dict(cfg=cfg, seed=seed, d=d, V=V, R=R, N=N, M=M,
               draft_tokens=draft, parents=parents, num_nodes=num_nodes,
               H_bits=H_bits, W_bits=W_bits, designated=designated.astype(np.int32), alpha_r=alpha_r)
    if gen_T:
        out["T_bits"] = gen_target_logits(rng, M, V, designated, cfg.inject_ties)
    return out


def gen_target_logits(rng: np.random.Generator, M: int, V: int, designated: np.ndarray,
                      inject_ties: bool = False) -> np.ndarray:
    T_bits = np.empty((M, V), dtype=np.uint16)
    step = max(1, (1 << 24) // V)
    for m0 in range(0, M, step):
        m1 = min(M, m0 + step)
        t = rng.standard_normal((m1 - m0, V), dtype=np.float32) * np.float32(2.0)
        rows = np.arange(m1 - m0)
        t[rows, designated[m0:m1]] = t.max(axis=1) + np.float32(1.0)
        T_bits[m0:m1] = f32_to_bf16_bits(t)
    if inject_ties:
        _inject_ties(rng, T_bits)
    return T_bits


def _inject_ties(rng: np.random.Generator, T_bits: np.ndarray) -> None:
    """Tiny config only: plant exact bf16 ties (PAPER silent; SPEC S:84/S:207
    lowest index wins) at the argmax, at the 10th place, and a +-0 pair."""
    M, V = T_bits.shape
    vals = bf16_bits_to_f32(T_bits)
    for m in range(0, M, 3):
        order = np.argsort(-vals[m], kind="stable")
        top = int(order[0])
        # tie at the argmax: copy the max to a random other column
        j = int(rng.integers(0, V))
        if j != top:
            T_bits[m, j] = T_bits[m, top]
        # tie at the 10th place: copy the 10th value onto the 11th-ranked column
        T_bits[m, int(order[10])] = T_bits[m, int(order[9])]
    # a +-0 pair on one row, placed at the very top of that row
    m = 1
    T_bits[m, :] = f32_to_bf16_bits(-np.abs(vals[m]) - 1.0)   # everything negative
    T_bits[m, 7] = 0x8000                                        # -0.0
    T_bits[m, 3] = 0x0000                                        # +0.0 (equal; lower index)


def gen_trace_topk(cfg: TraceConfig | str, K_t: int = 1024, seed: Optional[int] = None) -> dict:
    """NEXT F1 workload: the same trace (W, H, tokens, parents, planted designated tokens)
    with the verifier's logits delivered as the paper's transmitted payload — K_t
    (id, bf16 logit) pairs per row ("top-K = 1024").  Each row draws K_t
    distinct ids (the designated token always among them, at a random slot), logits
    ~ N(0, 2^2), and the designated token gets max + 1.0.  Drawn directly; nothing is
    selected from a dense row, so no method arithmetic lives here."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    tr = gen_trace(cfg, seed=seed, gen_T=False)
    rng = np.random.Generator(np.random.PCG64((cfg.seed if seed is None else seed) + 7919))
    M, V = tr["M"], tr["V"]
    K_t = min(K_t, V)
    ids = np.empty((M, K_t), dtype=np.int32)
    vals = np.empty((M, K_t), dtype=np.uint16)
    for m in range(M):
        row = rng.choice(V, size=K_t, replace=False)
        des = int(tr["designated"][m])
        hit = np.nonzero(row == des)[0]
        slot = int(hit[0]) if len(hit) else int(rng.integers(0, K_t))
        row[slot] = des
        v = rng.standard_normal(K_t, dtype=np.float32) * np.float32(2.0)
        v[slot] = v.max() + np.float32(1.0)
        ids[m] = row
        vals[m] = f32_to_bf16_bits(v)
    tr["Tk_idx"] = ids
    tr["Tk_bits"] = vals
    tr["K_t"] = K_t
    return tr


def gen_adamw_inputs(n: int, steps: int, seed: int = 4242, grad_scale: float = 1e-3) -> dict:
    """NEXT F3 inputs: fp32 master weights (the lm_head init of gen_trace, N(0, (2/sqrt d)^2)
    with d = 4096) and `steps` fp32 gradients ~ N(0, grad_scale^2).  Draws only."""
    rng = np.random.Generator(np.random.PCG64(seed))
    W = (rng.standard_normal(n, dtype=np.float32) * np.float32(2.0 / 64.0)).astype(np.float32)
    G = [(rng.standard_normal(n, dtype=np.float32) * np.float32(grad_scale)).astype(np.float32) for _ in range(steps)]
    return dict(W=W, G=G)


# ----------------------------------------------------------------------------- NEXT F4
@dataclasses.dataclass(frozen=True)
class TreeAttnConfig:
    """Tree-attention workload of the draft layer (F4): R requests, each a ragged prefix of
    P_r cached positions (K/V) plus the N + 1 tree rows (root + draft nodes)."""
    name: str
    R: int
    N: int
    Hq: int
    Hkv: int
    dh: int
    p_min: int
    p_max: int
    seed: int
    tree: bool = False
    beam: int = 4
    ragged_nodes: bool = False


TREE_ATTN_CONFIGS = {
    # oracle-pin sizes (not run on the GPU: dh != 128)
    "ta_tiny": TreeAttnConfig("ta_tiny", R=3, N=6, Hq=4, Hkv=2, dh=8, p_min=0, p_max=5, seed=3001, tree=True, beam=2),
    # GPU parity: several 64-key tiles, ragged tails, an empty prefix, ragged node counts
    "ta_small": TreeAttnConfig("ta_small", R=5, N=12, Hq=8, Hkv=2, dh=128, p_min=0, p_max=300, seed=3002,
                               tree=True, beam=3, ragged_nodes=True),
    "ta_chain": TreeAttnConfig("ta_chain", R=6, N=5, Hq=32, Hkv=8, dh=128, p_min=1, p_max=200, seed=3003),
    "ta_gqa8": TreeAttnConfig("ta_gqa8", R=4, N=15, Hq=16, Hkv=2, dh=128, p_min=60, p_max=130, seed=3004,
                              tree=True, beam=5),
    # full sizes: the Llama chain traces and the tree-draft traces (BASELINE configs[1], [4]);
    # Llama-3.1-8B / Qwen3-8B attention shapes (32 query heads, 8 KV heads, head_dim 128);
    # prefixes up to the paper's max sequence 2048 minus the tree depth
    "ta_llama": TreeAttnConfig("ta_llama", R=64, N=5, Hq=32, Hkv=8, dh=128, p_min=128, p_max=2042, seed=3011),
    "ta_tree": TreeAttnConfig("ta_tree", R=1024, N=24, Hq=32, Hkv=8, dh=128, p_min=128, p_max=2041, seed=3012,
                              tree=True, beam=4),
}


def gen_tree_attn_meta(cfg: TreeAttnConfig | str) -> dict:
    """Structure only: prefix lengths ~ U[p_min, p_max], the parent array (chain: None;
    tree: the same beam recipe as gen_trace) and ragged node counts."""
    if isinstance(cfg, str):
        cfg = TREE_ATTN_CONFIGS[cfg]
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    lens = rng.integers(cfg.p_min, cfg.p_max + 1, size=cfg.R).astype(np.int64)
    if cfg.R > 1 and cfg.p_min == 0:
        lens[1] = 0                                   # an empty prefix
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    parents = _tree_parents(rng, cfg.R, cfg.N // cfg.beam, cfg.beam) if cfg.tree else None
    num_nodes = None
    if cfg.ragged_nodes:
        num_nodes = np.full(cfg.R, cfg.N, dtype=np.int32)
        num_nodes[0] = max(1, cfg.N // 2)
        if cfg.R > 2:
            num_nodes[2] = 0
    return dict(cfg=cfg, prefix_off=off, parents=parents, num_nodes=num_nodes)


def gen_tree_attn(cfg: TreeAttnConfig | str, requests=None) -> dict:
    """Q [R, N+1, Hq, dh], Kt/Vt [R, N+1, Hkv, dh], Kp/Vp [P_total, Hkv, dh], dO like Q, as
    bf16 bits.  Each request draws from its own stream PCG64(seed * 100003 + 1 + r), so
    `requests` (a subset) reproduces exactly those requests' inputs (the full-size parity
    tests hand the oracle a sample).  Q, K ~ N(0, 1) (scaled scores ~ N(0, 1)); the query
    heads of every fourth KV group are scaled by 3 (peaked rows); V ~ N(0, 1); dO ~
    N(0, 0.1^2)."""
    meta = gen_tree_attn_meta(cfg)
    c = meta["cfg"]
    off = meta["prefix_off"]
    reqs = np.arange(c.R) if requests is None else np.asarray(requests)
    N1 = c.N + 1
    Q = np.empty((len(reqs), N1, c.Hq, c.dh), np.uint16)
    dO = np.empty_like(Q)
    Kt = np.empty((len(reqs), N1, c.Hkv, c.dh), np.uint16)
    Vt = np.empty_like(Kt)
    lens = [int(off[r + 1] - off[r]) for r in reqs]
    Kp = np.empty((sum(lens), c.Hkv, c.dh), np.uint16)
    Vp = np.empty_like(Kp)
    qscale = np.ones((c.Hq, 1), np.float32)
    G = c.Hq // c.Hkv
    for h in range(c.Hq):
        if (h // G) % 4 == 3:
            qscale[h] = 3.0
    pos = 0
    for i, r in enumerate(reqs):
        rng = np.random.Generator(np.random.PCG64(c.seed * 100003 + 1 + int(r)))
        Q[i] = f32_to_bf16_bits(rng.standard_normal((N1, c.Hq, c.dh), dtype=np.float32) * qscale)
        Kt[i] = f32_to_bf16_bits(rng.standard_normal((N1, c.Hkv, c.dh), dtype=np.float32))
        Vt[i] = f32_to_bf16_bits(rng.standard_normal((N1, c.Hkv, c.dh), dtype=np.float32))
        L = lens[i]
        Kp[pos:pos + L] = f32_to_bf16_bits(rng.standard_normal((L, c.Hkv, c.dh), dtype=np.float32))
        Vp[pos:pos + L] = f32_to_bf16_bits(rng.standard_normal((L, c.Hkv, c.dh), dtype=np.float32))
        dO[i] = f32_to_bf16_bits(rng.standard_normal((N1, c.Hq, c.dh), dtype=np.float32) * np.float32(0.1))
        pos += L
    sub_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    par = meta["parents"]
    nn = meta["num_nodes"]
    return dict(cfg=c, requests=reqs, Q_bits=Q, Kt_bits=Kt, Vt_bits=Vt, Kp_bits=Kp, Vp_bits=Vp, dO_bits=dO,
                prefix_off=sub_off, parents=None if par is None else par[reqs],
                num_nodes=None if nn is None else nn[reqs])

"""CPU oracle for NEXT row F4 (tree attention of the draft layer) — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
legs may import this module.  The product path (`libaurora.so` and its binding) never
imports, links or calls anything under `oracle/`, and this module imports nothing from it.

What it computes (PAPER.md = P, SPEC.md = S, line numbers):

  P:163-169 §3.2 "Efficient Tree Attention ... a custom attention mask that respects the
  causal structure of the speculative tree, we can process all accepted and rejected
  branches in a single batched forward and backward pass"; S:134-140 / S:166-174 (the
  tree: parents[n] < n, -1 = root).  Reading F4-R1..R5:

    rows of request r:  s = 0 is the root (the last verified context position),
                        s = n + 1 is draft node n (the same row order as the lm_head path);
    keys of request r:  the P_r prefix positions (K/V given, ragged lengths) followed by
                        the N + 1 tree rows;
    mask:               row s sees every prefix key and the tree rows in anc*(s), the
                        ancestor closure of s (its ancestors, the root and s itself);
                        rows of nodes n >= num_nodes[r] (ragged padding) are not keys of
                        anyone and, as queries, output 0 with lse = -inf.

  Per (request, head h, kv head h // G):
      S = scale * Q K^T + mask(-inf),  lse = log sum exp S,  P = exp(S - lse),  O = P V
  and the gradient of a scalar loss with dL/dO = dO (textbook softmax-attention backward):
      dV = P^T dO,  dP = dO V^T,  dS = P * (dP - rowsum(P * dP)),
      dQ = scale * dS K,  dK = scale * dS^T Q.
  GQA: the G = Hq / Hkv query heads of a kv head share its K, V; their dK, dV add up.

Tree positions and RoPE (F4-R6): node n of request r sits at position
P_r + depth(n) (depth of the root row = 0, a child of the root = 1, ...), so siblings share a
position; queries and tree keys are rotated there with the rotate-half convention used by the
Llama / Qwen3 targets, x'[i] = x[i] cos(p w_i) - x[i + dh/2] sin(p w_i),
x'[i + dh/2] = x[i + dh/2] cos(p w_i) + x[i] sin(p w_i), w_i = theta^(-2i/dh); the gradient
w.r.t. the unrotated input is the inverse (transposed) rotation.

Everything is float64 on the exact upcast of the bf16 inputs.  Pins:
tests/test_tree_attn_oracle.py (torch f64 SDPA + autograd with a mask built by boolean
matrix powers, causal special case, brute-force scalar loops, finite differences,
branch-independence, single-key identity, GQA = repeated-KV MHA; RoPE against transformers'
apply_rotary_pos_emb, rotation / inverse / relative-position invariants).
"""
from __future__ import annotations

import numpy as np


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    b = np.asarray(bits, dtype=np.uint16)
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def ancestor_rows(parents_r, num_nodes_r: int, N: int) -> list:
    """anc*(s) for every tree row s = 0..N (row 0 = root, row n+1 = node n), by walking
    parent pointers (S:129 parents[n] < n; -1 = child of the root).  parents_r None = chain
    (parent of node n is n - 1).  Rows of padded nodes (n >= num_nodes_r) get []."""
    out = [[0]]
    for n in range(N):
        if n >= num_nodes_r:
            out.append([])
            continue
        rows = [n + 1]
        p = (n - 1) if parents_r is None else int(parents_r[n])
        while p >= 0:
            rows.append(p + 1)
            p = (p - 1) if parents_r is None else int(parents_r[p])
        rows.append(0)
        out.append(sorted(rows))
    return out


def _keys(Kp, Vp, Kt, Vt, off, r, hk):
    p0, p1 = int(off[r]), int(off[r + 1])
    K = np.concatenate([Kp[p0:p1, hk, :], Kt[r, :, hk, :]], axis=0)
    V = np.concatenate([Vp[p0:p1, hk, :], Vt[r, :, hk, :]], axis=0)
    return K, V, p1 - p0


def _allowed(anc, Pr, N):
    """[N+1, Pr+N+1] boolean: prefix keys always, tree keys per anc*(s)."""
    A = np.zeros((N + 1, Pr + N + 1), dtype=bool)
    for s in range(N + 1):
        if anc[s]:
            A[s, :Pr] = True
            A[s, [Pr + t for t in anc[s]]] = True
    return A


def tree_attention_fwd(Q, Kt, Vt, Kp, Vp, prefix_off, parents=None, num_nodes=None, scale=None):
    """Q [R, N+1, Hq, dh], Kt/Vt [R, N+1, Hkv, dh], Kp/Vp [P_total, Hkv, dh] (float64),
    prefix_off [R+1].  Returns O [R, N+1, Hq, dh], lse [R, N+1, Hq] (natural log; -inf on
    padded rows)."""
    R, N1, Hq, dh = Q.shape
    N = N1 - 1
    Hkv = Kt.shape[2]
    G = Hq // Hkv
    scale = 1.0 / np.sqrt(dh) if scale is None else scale
    O = np.zeros_like(Q)
    lse = np.full((R, N1, Hq), -np.inf)
    for r in range(R):
        nn = N if num_nodes is None else int(num_nodes[r])
        anc = ancestor_rows(None if parents is None else parents[r], nn, N)
        for h in range(Hq):
            K, V, Pr = _keys(Kp, Vp, Kt, Vt, prefix_off, r, h // G)
            A = _allowed(anc, Pr, N)
            S = scale * (Q[r, :, h, :] @ K.T)
            for s in range(N1):
                if not anc[s]:
                    continue
                x = S[s, A[s]]
                mx = x.max()
                l = mx + np.log(np.sum(np.exp(x - mx)))
                p = np.exp(x - l)
                O[r, s, h, :] = p @ V[A[s]]
                lse[r, s, h] = l
    return O, lse


def tree_attention_bwd(Q, Kt, Vt, Kp, Vp, prefix_off, dO, parents=None, num_nodes=None, scale=None):
    """Gradients of <dO, O> wrt Q, Kt, Vt, Kp, Vp (float64, same shapes as the inputs)."""
    R, N1, Hq, dh = Q.shape
    N = N1 - 1
    Hkv = Kt.shape[2]
    G = Hq // Hkv
    scale = 1.0 / np.sqrt(dh) if scale is None else scale
    dQ = np.zeros_like(Q)
    dKt, dVt = np.zeros_like(Kt), np.zeros_like(Vt)
    dKp, dVp = np.zeros_like(Kp), np.zeros_like(Vp)
    for r in range(R):
        nn = N if num_nodes is None else int(num_nodes[r])
        anc = ancestor_rows(None if parents is None else parents[r], nn, N)
        p0, p1 = int(prefix_off[r]), int(prefix_off[r + 1])
        for h in range(Hq):
            hk = h // G
            K, V, Pr = _keys(Kp, Vp, Kt, Vt, prefix_off, r, hk)
            A = _allowed(anc, Pr, N)
            S = scale * (Q[r, :, h, :] @ K.T)
            S = np.where(A, S, -np.inf)
            P = np.zeros_like(S)
            for s in range(N1):
                if anc[s]:
                    x = S[s, A[s]]
                    P[s, A[s]] = np.exp(x - x.max()) / np.sum(np.exp(x - x.max()))
            dOh = dO[r, :, h, :]
            dV = P.T @ dOh
            dP = dOh @ V.T
            dS = P * (dP - np.sum(P * dP, axis=1, keepdims=True))
            dQ[r, :, h, :] = scale * (dS @ K)
            dK = scale * (dS.T @ Q[r, :, h, :])
            dKp[p0:p1, hk, :] += dK[:Pr]
            dVp[p0:p1, hk, :] += dV[:Pr]
            dKt[r, :, hk, :] += dK[Pr:]
            dVt[r, :, hk, :] += dV[Pr:]
    return dQ, dKt, dVt, dKp, dVp


def from_inputs(inp: dict):
    """Upcast a tracegen.gen_tree_attn() record to the oracle's float64 arguments."""
    f = bf16_bits_to_f64
    return dict(Q=f(inp["Q_bits"]), Kt=f(inp["Kt_bits"]), Vt=f(inp["Vt_bits"]), Kp=f(inp["Kp_bits"]),
                Vp=f(inp["Vp_bits"]), prefix_off=inp["prefix_off"], parents=inp["parents"],
                num_nodes=inp["num_nodes"])


def fwd_bwd(inp: dict, requests=None):
    """O, lse and all gradients for a generated record (optionally a subset of requests:
    each request is independent, so a sample is exact for the rows it covers)."""
    a = from_inputs(inp)
    dO = bf16_bits_to_f64(inp["dO_bits"])
    if requests is not None:
        a, dO = _select(a, dO, requests)
    O, lse = tree_attention_fwd(**a)
    grads = tree_attention_bwd(dO=dO, **a)
    return dict(O=O, lse=lse, dQ=grads[0], dKt=grads[1], dVt=grads[2], dKp=grads[3], dVp=grads[4],
                prefix_off=a["prefix_off"])


def _select(a, dO, reqs):
    reqs = np.asarray(reqs)
    off = a["prefix_off"]
    pieces = [np.arange(off[r], off[r + 1]) for r in reqs]
    pidx = np.concatenate(pieces) if pieces else np.zeros(0, np.int64)
    lens = np.array([off[r + 1] - off[r] for r in reqs])
    b = dict(Q=a["Q"][reqs], Kt=a["Kt"][reqs], Vt=a["Vt"][reqs], Kp=a["Kp"][pidx], Vp=a["Vp"][pidx],
             prefix_off=np.concatenate([[0], np.cumsum(lens)]).astype(np.int64),
             parents=None if a["parents"] is None else a["parents"][reqs],
             num_nodes=None if a["num_nodes"] is None else a["num_nodes"][reqs])
    return b, dO[reqs]


def tree_positions(parents_r, num_nodes_r: int, N: int, P_r: int) -> np.ndarray:
    """Position of every tree row (F4-R6): P_r + depth, depth by walking parent pointers;
    rows of padded nodes get -1 (left unrotated)."""
    pos = np.full(N + 1, -1, dtype=np.int64)
    pos[0] = P_r
    for n in range(min(num_nodes_r, N)):
        d, p = 1, (n - 1) if parents_r is None else int(parents_r[n])
        while p >= 0:
            d += 1
            p = (p - 1) if parents_r is None else int(parents_r[p])
        pos[n + 1] = P_r + d
    return pos


def rope(x: np.ndarray, pos: np.ndarray, theta: float, inverse: bool = False) -> np.ndarray:
    """Rotate-half RoPE of x [..., rows, heads, dh] at integer positions pos [..., rows]
    (pos < 0: row left unchanged); inverse=True applies the transposed rotation."""
    dh = x.shape[-1]
    half = dh // 2
    w = theta ** (-2.0 * np.arange(half, dtype=np.float64) / dh)
    ang = np.asarray(pos, dtype=np.float64)[..., None, None] * w          # [..., rows, 1, half]
    c, s_ = np.cos(ang), np.sin(ang)
    if inverse:
        s_ = -s_
    a, b = x[..., :half], x[..., half:]
    out = np.concatenate([a * c - b * s_, b * c + a * s_], axis=-1)
    keep = np.asarray(pos)[..., None, None] < 0
    return np.where(keep, x, out)


def tree_rope_positions(prefix_off, parents, num_nodes, R: int, N: int) -> np.ndarray:
    """[R, N+1] positions of every tree row of the batch."""
    out = np.empty((R, N + 1), dtype=np.int64)
    for r in range(R):
        nn = N if num_nodes is None else int(num_nodes[r])
        out[r] = tree_positions(None if parents is None else parents[r], nn, N, int(prefix_off[r + 1] - prefix_off[r]))
    return out

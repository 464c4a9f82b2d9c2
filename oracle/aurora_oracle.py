"""CPU oracle for the Aurora speculator-training hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this module.  The product path (the CUDA
library `libaurora.so` and its Python binding) never imports, links or calls
anything under `oracle/`, and this module imports nothing from the product.

It is the plain, slow, float64 definition of what the path computes, written
step by step in the paper's order (PAPER.md = P, SPEC.md = S, line numbers):

  O1 target_scan   y = argmax of the verifier logits (lowest index wins ties),
                   and the top-K list ordered by (value desc, index asc).
                   target_scan_topk: the same over the transmitted top-K payload (F1).
                   P:120 §2.1 "accepting the longest matching prefix" (greedy,
                   P:526 Table 3 "Top-k Sampling 1"); ties S:84.
  O2 verify        acc(n) = acc(parent(n)) AND [x_n == y at the parent's row];
                   accept_len = (#accepted) + 1 (bonus counts);
                   bonus = y at the deepest accepted row.  P:120.
  O3 row_targets   ACCEPT rows (root + accepted nodes) use the target's top-k_acc
                   support, DISCARD rows (context contains a rejected token)
                   the top-k_disc support (k=10); p~ = target
                   softmax renormalised on the support; weight 1/N_A or
                   lambda/N_D (lambda=1.0; per-term means).
  O4 loss_fwd      L = sum_m w_m KL(p~_m || softmax(z_m)),  z_m = W h_m
                   (Eq. 3; full-vocab log-softmax per north_star).
  O5 loss_bwd      dL/dz = w (q - p~) (gradient of KL(p~||q) wrt logits);
                   dW = dZ^T H, dH = dZ W (fp32 gradients; here fp64).
  O6 step_variants (NEXT F2, the objectives of §5.1, and SPEC's restricted-softmax
                   discard loss S:328-331): accepted rows with
                   reverse KL(q || p_target) (gradient q*((ln q - ln p) - KL))
                   plus beta * NTP cross-entropy on the verified token,
                   discard rows with the unfiltered dense KL(p_target || q) ("top-k =
                   0").  Written directly from those definitions on
                   full-vocabulary rows (no decomposition shared with the kernels).
  O7 adamw_step    (NEXT F3) one AdamW step (Table 3): global-norm clip at
                   0.5, linear warm-up over 400 steps then constant, decoupled
                   weight decay, bias-corrected moments (SPEC: betas 0.9/0.999, eps 1e-8).

Readings where the paper is silent/ambiguous are listed in DESIGN.md
("Readings Q1-Q15"); each function names the ones it relies on.

Pins (tests/test_oracle_pins.py, `-m "not gpu"`): brute-force top-k on tiny
vocabularies and hand-written tie rows (tests/golden), SPEC worked examples
S:182-184 / S:325 / S:345, exhaustive chain and tree verification
enumeration, Eq. 1 Monte Carlo, torch f64 cross_entropy / kl_div /
autograd, central finite differences, row-sum-zero and shift invariance.
"""
from __future__ import annotations

import numpy as np

ACCEPT, DISCARD, PAD = 0, 1, 2


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    """Exact upcast of bf16 bit patterns: bf16 -> f32 by a 16-bit shift -> f64."""
    b = np.asarray(bits, dtype=np.uint16)
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


# --------------------------------------------------------------------------- O1
def target_scan(T_rows: np.ndarray, k_max: int):
    """O1 (reading Q8).

    T_rows: f64 [m, V].  Returns (argmax int64 [m], topk int64 [m, k_max],
    nonfinite bool).  Order is (value desc, index asc) with numeric compare, so
    -0 == +0; a stable argsort of -t gives exactly that order.
    """
    T_rows = np.asarray(T_rows, dtype=np.float64)
    nonfinite = not bool(np.all(np.isfinite(T_rows)))
    order = np.argsort(-T_rows, axis=1, kind="stable")
    topk = order[:, :k_max]
    return topk[:, 0].copy(), topk.copy(), nonfinite


def target_scan_topk(idx: np.ndarray, val: np.ndarray, k_max: int, V: int):
    """O1' (NEXT F1): the same scan over the paper's transmitted sparse payload — the
    target's top-K logits per position as (global id, logit) pairs ("top-K
    logits filtering (e.g., K=1024)"; SPEC S:420-428 compressed payload).  The order is
    again (value desc, index asc) over the transmitted pairs.

    idx int [m, K_t], val f64 [m, K_t].  Returns (argmax [m], topk ids [m, k_max],
    nonfinite, out_of_range, duplicate) — the last three are the conditions the kernel
    reports in the status word.
    """
    idx = np.asarray(idx, dtype=np.int64)
    val = np.asarray(val, dtype=np.float64)
    nonfinite = not bool(np.all(np.isfinite(val)))
    out_of_range = bool(np.any((idx < 0) | (idx >= V)))
    dup = any(len(np.unique(r)) != len(r) for r in idx)
    topk = np.empty((idx.shape[0], k_max), dtype=np.int64)
    for m in range(idx.shape[0]):
        order = np.lexsort((idx[m], -val[m]))       # primary: value desc, secondary: id asc
        topk[m] = idx[m][order[:k_max]]
    return topk[:, 0].copy(), topk, nonfinite, out_of_range, dup


# --------------------------------------------------------------------------- O2
def verify(draft_tokens: np.ndarray, parents, num_nodes, argmax: np.ndarray,
           discard_scope: int = 0):
    """O2 greedy verification over chains or trees.

    Row of node n in request r is r*(N+1) + n + 1; the root row is r*(N+1).
    Node n is *matched* iff draft_tokens[r,n] == argmax[row(parent(n))]; it is
    *accepted* iff matched and its parent is accepted (root always is).  If two
    siblings both match, the lowest node index wins (reading Q12; "the
    accepted path is a path, never a branch").
    accept_len = #accepted + 1 ("accepted_path length + 1").
    bonus = argmax at the row of the deepest accepted node (root row if none).
    Row classes (readings Q1-Q3): root and accepted-node rows ACCEPT; other
    valid node rows DISCARD ("all rejected nodes"); with discard_scope=1
    only first-divergence rows (rejected node whose parent is accepted) stay
    DISCARD and deeper ones become PAD; nodes >= num_nodes[r] are PAD.
    """
    draft_tokens = np.asarray(draft_tokens)
    R, N = draft_tokens.shape
    accepted = np.zeros((R, N), dtype=np.uint8)
    accept_len = np.zeros(R, dtype=np.int32)
    bonus = np.zeros(R, dtype=np.int32)
    row_class = np.full(R * (N + 1), PAD, dtype=np.uint8)
    for r in range(R):
        nn = N if num_nodes is None else int(num_nodes[r])
        base = r * (N + 1)
        acc = [False] * N
        depth = [0] * N
        won_parent = set()            # parents that already have an accepted child
        for n in range(nn):
            p = (n - 1) if parents is None else int(parents[r, n])
            if not (-1 <= p < n):
                raise ValueError("malformed parents: parent must satisfy -1 <= p < n")
            parent_acc = True if p < 0 else acc[p]
            depth[n] = 1 if p < 0 else depth[p] + 1
            match = int(draft_tokens[r, n]) == int(argmax[base + p + 1])
            if parent_acc and match and p not in won_parent:
                acc[n] = True
                won_parent.add(p)
        row_class[base] = ACCEPT
        deepest_row, deepest_depth, a = 0, 0, 0
        for n in range(nn):
            p = (n - 1) if parents is None else int(parents[r, n])
            if acc[n]:
                accepted[r, n] = 1
                row_class[base + n + 1] = ACCEPT
                a += 1
                if depth[n] > deepest_depth:
                    deepest_row, deepest_depth = n + 1, depth[n]
            else:
                first_div = (p < 0) or acc[p]
                if discard_scope == 0 or first_div:
                    row_class[base + n + 1] = DISCARD
        accept_len[r] = a + 1
        bonus[r] = int(argmax[base + deepest_row])
    return dict(accepted=accepted, accept_len=accept_len, bonus=bonus, row_class=row_class)


# --------------------------------------------------------------------------- O3
def row_targets(row_class: np.ndarray, T_rows_by_m, topk: np.ndarray, k_accept: int = 1,
                k_discard: int = 10, lambda_discard: float = 1.0, normalize: int = 0,
                rows=None):
    """O3 row supports, renormalised target distributions and weights.

    P:185 (accepted term: CE on the verified token = support {y} when
    k_accept=1, reading Q5), P:191-195 (discard term, top-k filtered target,
    k=10 P:520, lambda=1.0 P:521), reading Q6 (support = target top-k by
    (logit desc, index asc), target renormalised on it), reading Q7 (per-term
    means over the global counts N_A, N_D; normalize=1: mean over all rows).

    T_rows_by_m(m) -> f64 [V] gives the verifier logits of row m; topk[m] is O1's
    ordered list.  Returns dict with per-row lists sup_idx (index-sorted),
    sup_p (aligned), H (sum p log p), w, and counts (N_A, N_D).
    """
    M = row_class.shape[0]
    n_acc = int(np.sum(row_class == ACCEPT))
    n_dis = int(np.sum(row_class == DISCARD))
    rows = range(M) if rows is None else rows
    sup_idx, sup_p, Hs, ws = {}, {}, {}, {}
    for m in rows:
        c = int(row_class[m])
        if c == PAD:
            sup_idx[m] = np.zeros(0, dtype=np.int64)
            sup_p[m] = np.zeros(0)
            Hs[m] = 0.0
            ws[m] = 0.0
            continue
        k = k_accept if c == ACCEPT else k_discard
        S = np.asarray(topk[m][:k], dtype=np.int64)
        t = np.asarray(T_rows_by_m(m), dtype=np.float64)[S]
        e = np.exp(t - t.max())
        p = e / e.sum()
        order = np.argsort(S, kind="stable")
        sup_idx[m] = S[order]
        sup_p[m] = p[order]
        Hs[m] = float(np.sum(p * np.log(p)))
        if normalize == 0:
            ws[m] = (1.0 / n_acc) if c == ACCEPT else (lambda_discard / n_dis if n_dis else 0.0)
        else:
            ws[m] = (1.0 if c == ACCEPT else lambda_discard) / (n_acc + n_dis)
    return dict(sup_idx=sup_idx, sup_p=sup_p, H=Hs, w=ws, counts=(n_acc, n_dis))


# --------------------------------------------------------------------------- O4
def logits(H64: np.ndarray, W_bits_or_64, v0: int, v1: int) -> np.ndarray:
    W = W_bits_or_64[v0:v1]
    if W.dtype == np.uint16:
        W = bf16_bits_to_f64(W)
    return H64 @ W.T


def loss_fwd(H64: np.ndarray, W, targets: dict, rows=None, chunk: int = 8192):
    """O4: per-row lse (exact f64 log-sum-exp over the full vocabulary),
    u_m = sum_{j in S_m} p~_j z_mj computed from direct dot products
    H_m . W_j, row loss l_m = lse_m - u_m + H~_m = KL(p~_m || q_m), and
    L = sum_m w_m l_m (Eq. 3)."""
    M = H64.shape[0]
    rows = np.arange(M) if rows is None else np.asarray(rows)
    Hr = H64[rows]
    V = W.shape[0]
    mx = np.full(len(rows), -np.inf)
    s = np.zeros(len(rows))
    for v0 in range(0, V, chunk):
        z = logits(Hr, W, v0, min(V, v0 + chunk))
        cm = z.max(axis=1)
        nm = np.maximum(mx, cm)
        s = s * np.exp(mx - nm) + np.exp(z - nm[:, None]).sum(axis=1)
        mx = nm
    lse = mx + np.log(s)
    row_loss = np.zeros(len(rows))
    for i, m in enumerate(rows):
        S = targets["sup_idx"][int(m)]
        if len(S) == 0:
            continue
        Ws = W[S]
        if Ws.dtype == np.uint16:
            Ws = bf16_bits_to_f64(Ws)
        zS = Ws @ H64[m]
        u = float(np.dot(targets["sup_p"][int(m)], zS))
        row_loss[i] = lse[i] - u + targets["H"][int(m)]
    w = np.array([targets["w"][int(m)] for m in rows])
    return dict(rows=rows, lse=lse, row_loss=row_loss, loss=float(np.dot(w, row_loss)))


# --------------------------------------------------------------------------- O5
def loss_bwd(H64: np.ndarray, W, targets: dict, lse: np.ndarray, g: float = 1.0,
             chunk: int = 8192, want_dW: bool = True):
    """O5: dZ = g w (softmax(z) - p~) on the support (S:321 FKL grad q - p),
    dW = dZ^T H, dH = dZ W.  Chunked over the vocabulary only to bound RAM
    (no recompute trick, no reordering of the sums beyond the chunking)."""
    M, d = H64.shape
    V = W.shape[0]
    w = np.array([targets["w"][m] for m in range(M)])
    dH = np.zeros((M, d))
    dW = np.zeros((V, d)) if want_dW else None
    for v0 in range(0, V, chunk):
        v1 = min(V, v0 + chunk)
        Wc = W[v0:v1]
        if Wc.dtype == np.uint16:
            Wc = bf16_bits_to_f64(Wc)
        z = H64 @ Wc.T
        dZ = np.exp(z - lse[:, None]) * (g * w)[:, None]
        for m in range(M):
            S = targets["sup_idx"][m]
            if len(S) == 0:
                continue
            sel = (S >= v0) & (S < v1)
            dZ[m, S[sel] - v0] -= g * w[m] * targets["sup_p"][m][sel]
        dH += dZ @ Wc
        if want_dW:
            dW[v0:v1] = dZ.T @ H64
    return dict(dH=dH, dW=dW)


def loss_bwd_sampled(H64: np.ndarray, W, targets: dict, lse: np.ndarray, dh_rows, dw_ranges, g: float = 1.0):
    """O5 restricted to what a full-size check can afford: dH at the rows `dh_rows`
    (dH_m = sum_j dz_mj W_j over the whole vocabulary) and dW at the vocabulary ranges
    `dw_ranges` (dW_j = sum_m dz_mj H_m over every row), with dz = g w (softmax(z) - p~)
    as in loss_bwd.  lse: f64 [M] for every row (O4).  Returns
    dict(dH=[len(dh_rows), d], dW={(v0, v1): [v1 - v0, d]})."""
    M, d = H64.shape
    w = np.array([targets["w"][m] for m in range(M)])
    Wf = lambda v0, v1: bf16_bits_to_f64(W[v0:v1]) if W.dtype == np.uint16 else W[v0:v1]

    def dz_block(rows, v0, v1):
        z = H64[rows] @ Wf(v0, v1).T
        dz = np.exp(z - lse[rows][:, None]) * (g * w[rows])[:, None]
        for i, m in enumerate(rows):
            S = targets["sup_idx"][int(m)]
            sel = (S >= v0) & (S < v1)
            dz[i, S[sel] - v0] -= g * w[m] * targets["sup_p"][int(m)][sel]
        return dz

    rows = np.asarray(dh_rows, dtype=np.int64)
    V = W.shape[0]
    dH = np.zeros((len(rows), d))
    for v0 in range(0, V, 8192):
        v1 = min(V, v0 + 8192)
        dH += dz_block(rows, v0, v1) @ Wf(v0, v1)
    dW = {}
    allrows = np.arange(M)
    for v0, v1 in dw_ranges:
        dW[(v0, v1)] = dz_block(allrows, v0, v1).T @ H64
    return dict(dH=dH, dW=dW)


def dlogits_rows(H64, W, targets, lse_rows, rows, g: float = 1.0):
    """Full dZ rows for a handful of rows (test hook counterpart)."""
    Wf = bf16_bits_to_f64(W) if W.dtype == np.uint16 else W
    out = []
    for i, m in enumerate(rows):
        z = Wf @ H64[m]
        dz = np.exp(z - lse_rows[i]) * g * targets["w"][m]
        S = targets["sup_idx"][m]
        dz[S] -= g * targets["w"][m] * targets["sup_p"][m]
        out.append(dz)
    return np.array(out)


# ------------------------------------------------------------------ whole step
def step(trace: dict, k_accept: int = 1, k_discard: int = 10, lambda_discard: float = 1.0,
         normalize: int = 0, discard_scope: int = 0, g: float = 1.0, want_grads: bool = True,
         want_dW: bool = True):
    """verify -> targets -> fwd -> bwd for one trace batch (everything f64)."""
    T = bf16_bits_to_f64(trace["T_bits"])
    H64 = bf16_bits_to_f64(trace["H_bits"])
    Wb = trace["W_bits"]
    k_max = max(k_accept, k_discard)
    amax, topk, nonfinite = target_scan(T, k_max)
    if nonfinite:
        raise ValueError("non-finite target logits")
    lab = verify(trace["draft_tokens"], trace["parents"], trace["num_nodes"], amax, discard_scope)
    tg = row_targets(lab["row_class"], lambda m: T[m], topk, k_accept, k_discard, lambda_discard, normalize)
    fw = loss_fwd(H64, Wb, tg)
    out = dict(argmax=amax, topk=topk, **lab, targets=tg, lse=fw["lse"], row_loss=fw["row_loss"],
               loss=fw["loss"])
    if want_grads:
        out.update(loss_bwd(H64, Wb, tg, fw["lse"], g=g, want_dW=want_dW))
    return out


def step_topk(trace: dict, k_accept: int = 1, k_discard: int = 10, lambda_discard: float = 1.0,
              normalize: int = 0, discard_scope: int = 0, g: float = 1.0, want_grads: bool = True):
    """verify -> targets -> fwd -> bwd with the sparse target payload (F1): trace holds
    Tk_idx int32 [M, K_t] and Tk_bits bf16 [M, K_t] instead of T_bits."""
    vals = bf16_bits_to_f64(trace["Tk_bits"])
    idx = np.asarray(trace["Tk_idx"], dtype=np.int64)
    H64 = bf16_bits_to_f64(trace["H_bits"])
    k_max = max(k_accept, k_discard)
    amax, topk, nonfinite, oor, dup = target_scan_topk(idx, vals, k_max, trace["V"])
    if nonfinite or oor or dup:
        raise ValueError("invalid sparse target payload")
    lab = verify(trace["draft_tokens"], trace["parents"], trace["num_nodes"], amax, discard_scope)

    def row_logits(m):  # the support values come from the transmitted pairs
        full = np.full(trace["V"], -np.inf)
        full[idx[m]] = vals[m]
        return full

    tg = row_targets(lab["row_class"], row_logits, topk, k_accept, k_discard, lambda_discard, normalize)
    fw = loss_fwd(H64, trace["W_bits"], tg)
    out = dict(argmax=amax, topk=topk, **lab, targets=tg, lse=fw["lse"], row_loss=fw["row_loss"], loss=fw["loss"])
    if want_grads:
        out.update(loss_bwd(H64, trace["W_bits"], tg, fw["lse"], g=g))
    return out


# --------------------------------------------------------------------------- O6
def _log_softmax(x: np.ndarray) -> np.ndarray:
    m = x.max()
    return x - (m + np.log(np.exp(x - m).sum()))


def step_variants(trace: dict, accept_loss: str = "fkl", ntp_beta: float = 0.0, k_accept: int = 1,
                  k_discard: int = 10, lambda_discard: float = 1.0, normalize: int = 0, discard_scope: int = 0,
                  g: float = 1.0, want_grads: bool = True, rows=None, discard_loss: str = "full"):
    """O6 (NEXT F2): the §5.1 objectives on a dense trace, row by row.

    ACCEPT rows: accept_loss "fkl" = KL(p~ || q) on the target top-k_accept support
    (Eq. 3, as O3-O5); "rkl" = KL(q || p) with p = softmax(T_row) over the full
    vocabulary (loss sum_j q_j (ln q_j - ln p_j), gradient q*((ln q - ln p) -
    KL)), plus ntp_beta * (-ln q_y) with y the verified token (gradient
    q - e_y; "RKL + NTP").  DISCARD rows: k_discard >= 1 = the filtered KL of
    O3-O5; k_discard = 0 = KL(p || q) over the full vocabulary ("top-k = 0", P:292,
    S:330 "topk=0 disables filtering"; gradient q - p).  Row weights as O3 (per-term
    means over the global counts, reading Q7); the NTP term shares the accepted rows'
    weight.  rows: subset of rows to evaluate (weights still use the full counts);
    gradients then cover only those rows' contributions.  discard_loss "restricted" (SPEC
    S:328-331, discard_loss_grad): on DISCARD rows with k_discard >= 1 both distributions are
    renormalised over the support, KL(p~ || q~) with q~ = softmax of the restricted logits z_S;
    the gradient is q~ - p~ on S and zero outside it.
    """
    T = bf16_bits_to_f64(trace["T_bits"])
    H64 = bf16_bits_to_f64(trace["H_bits"])
    W64 = bf16_bits_to_f64(trace["W_bits"])
    k_max = max(k_accept, k_discard, 1)
    amax, topk, nonfinite = target_scan(T, k_max)
    if nonfinite:
        raise ValueError("non-finite target logits")
    lab = verify(trace["draft_tokens"], trace["parents"], trace["num_nodes"], amax, discard_scope)
    cls = lab["row_class"]
    n_acc = int(np.sum(cls == ACCEPT))
    n_dis = int(np.sum(cls == DISCARD))
    M, d = H64.shape
    rows = range(M) if rows is None else rows
    row_loss = np.zeros(M)
    w = np.zeros(M)
    dH = np.zeros((M, d)) if want_grads else None
    dW = np.zeros_like(W64) if want_grads else None
    for m in rows:
        c = int(cls[m])
        if c == PAD:
            continue
        if normalize == 0:
            w[m] = (1.0 / n_acc) if c == ACCEPT else (lambda_discard / n_dis if n_dis else 0.0)
        else:
            w[m] = (1.0 if c == ACCEPT else lambda_discard) / (n_acc + n_dis)
        z = W64 @ H64[m]
        logq = _log_softmax(z)
        q = np.exp(logq)
        logp = _log_softmax(T[m])
        p = np.exp(logp)
        if c == ACCEPT and accept_loss == "rkl":
            kl = float(np.sum(q * (logq - logp)))
            grad = q * ((logq - logp) - kl)
            y = int(amax[m])
            loss = kl + ntp_beta * (-logq[y])
            grad = grad + ntp_beta * q
            grad[y] -= ntp_beta
        elif c == DISCARD and k_discard == 0:
            loss = float(np.sum(p * (logp - logq)))
            grad = q - p
        elif c == DISCARD and discard_loss == "restricted":
            S = np.asarray(topk[m][:k_discard], dtype=np.int64)
            pt = np.exp(_log_softmax(T[m][S]))
            logqt = _log_softmax(z[S])
            loss = float(np.sum(pt * (np.log(pt) - logqt)))
            grad = np.zeros_like(q)
            grad[S] = np.exp(logqt) - pt
        else:
            k = k_accept if c == ACCEPT else k_discard
            S = np.asarray(topk[m][:k], dtype=np.int64)
            pt = np.exp(_log_softmax(T[m][S]))
            loss = float(np.sum(pt * (np.log(pt) - logq[S])))
            grad = q.copy()
            grad[S] -= pt
        row_loss[m] = loss
        if want_grads:
            dz = g * w[m] * grad
            dH[m] = dz @ W64
            dW += np.outer(dz, H64[m])
    out = dict(argmax=amax, topk=topk, **lab, w=w, row_loss=row_loss, loss=float(np.dot(w, row_loss)),
               counts=(n_acc, n_dis))
    if want_grads:
        out.update(dH=dH, dW=dW)
    return out


# --------------------------------------------------------------------------- O7
def warmup_lr(lr: float, step: int, warmup_steps: int) -> float:
    """S:379 'Learning rate at step s < 400 equals base_lr*s/400; afterwards constant'."""
    return lr * step / warmup_steps if (warmup_steps > 0 and step < warmup_steps) else lr


def adamw_step(W: np.ndarray, m: np.ndarray, v: np.ndarray, dW: np.ndarray, step: int, lr: float,
               beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8, weight_decay: float = 0.0,
               max_grad_norm: float = 0.5, warmup_steps: int = 400, extra_sq: float = 0.0):
    """O7 (NEXT F3): AdamW (Loshchilov & Hutter: decoupled weight decay) with global-norm
    clipping, in the paper's order: norm = sqrt(sum g^2 (+ other groups));
    g <- g * min(1, max_norm / (norm + 1e-6)); m <- b1 m + (1-b1) g; v <- b2 v + (1-b2) g^2;
    W <- W - lr_t (m/(1-b1^t) / (sqrt(v/(1-b2^t)) + eps) + wd W).  f64; returns new arrays
    and the pre-clip norm."""
    W = np.asarray(W, dtype=np.float64)
    m = np.asarray(m, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    g = np.asarray(dW, dtype=np.float64)
    norm = float(np.sqrt(np.sum(g * g) + extra_sq))
    clip = min(1.0, max_grad_norm / (norm + 1e-6)) if max_grad_norm > 0 else 1.0
    g = g * clip
    lr_t = warmup_lr(lr, step, warmup_steps)
    m = beta1 * m + (1.0 - beta1) * g
    v = beta2 * v + (1.0 - beta2) * g * g
    mhat = m / (1.0 - beta1 ** step)
    vhat = v / (1.0 - beta2 ** step)
    W = W - lr_t * (mhat / (np.sqrt(vhat) + eps) + weight_decay * W)
    return W, m, v, norm

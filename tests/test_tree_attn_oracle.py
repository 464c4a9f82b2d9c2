"""Pins for the F4 tree-attention oracle (oracle/tree_attention.py) against things other
than itself (-m "not gpu"): torch f64 scaled_dot_product_attention + autograd with a mask
built a different way (boolean matrix powers of the parent adjacency), the causal special
case (a chain with no prefix is plain causal attention), brute-force scalar loops, central
finite differences, branch independence (every branch in one pass without
seeing its siblings), the single-key identity and GQA = MHA with repeated K/V.
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import tree_attention as TA
import tracegen


def _inputs(name="ta_tiny"):
    inp = tracegen.gen_tree_attn(name)
    return inp, TA.from_inputs(inp), TA.bf16_bits_to_f64(inp["dO_bits"])


def _closure_mask(parents_r, num_nodes_r, N):
    """Ancestor closure by boolean matrix powers: A[s, t] = t is the parent row of s (or
    s itself); closure = (I + A)^(N+1) > 0.  Independent of the oracle's pointer walk."""
    N1 = N + 1
    A = torch.zeros(N1, N1, dtype=torch.float64)
    for n in range(min(num_nodes_r, N)):
        p = (n - 1) if parents_r is None else int(parents_r[n])
        A[n + 1, p + 1] = 1.0
    C = torch.eye(N1, dtype=torch.float64)
    step = torch.eye(N1, dtype=torch.float64) + A
    for _ in range(N1):
        C = (C @ step).clamp(max=1.0)
    M = C > 0
    valid = torch.zeros(N1, dtype=torch.bool)
    valid[0] = True
    valid[1:min(num_nodes_r, N) + 1] = True
    return M & valid[:, None] & valid[None, :], valid


def _torch_ref(a, dO):
    """Per request: SDPA over [prefix; tree] keys with the closure mask; autograd grads."""
    R, N1, Hq, dh = a["Q"].shape
    N = N1 - 1
    Hkv = a["Kt"].shape[2]
    G = Hq // Hkv
    off = a["prefix_off"]
    out = dict(O=np.zeros_like(a["Q"]), lse=np.full((R, N1, Hq), -np.inf), dQ=np.zeros_like(a["Q"]),
               dKt=np.zeros_like(a["Kt"]), dVt=np.zeros_like(a["Vt"]),
               dKp=np.zeros_like(a["Kp"]), dVp=np.zeros_like(a["Vp"]))
    for r in range(R):
        nn = N if a["num_nodes"] is None else int(a["num_nodes"][r])
        tm, valid = _closure_mask(None if a["parents"] is None else a["parents"][r], nn, N)
        p0, p1 = int(off[r]), int(off[r + 1])
        Pr = p1 - p0
        mask = torch.cat([valid[:, None].expand(N1, Pr), tm], dim=1)          # [N1, Pr + N1]
        q = torch.tensor(a["Q"][r].transpose(1, 0, 2), requires_grad=True)    # [Hq, N1, dh]
        kp = torch.tensor(a["Kp"][p0:p1].transpose(1, 0, 2), requires_grad=True)
        vp = torch.tensor(a["Vp"][p0:p1].transpose(1, 0, 2), requires_grad=True)
        kt = torch.tensor(a["Kt"][r].transpose(1, 0, 2), requires_grad=True)
        vt = torch.tensor(a["Vt"][r].transpose(1, 0, 2), requires_grad=True)
        k = torch.cat([kp, kt], dim=1).repeat_interleave(G, dim=0)
        v = torch.cat([vp, vt], dim=1).repeat_interleave(G, dim=0)
        vq = valid.nonzero().flatten()
        o = F.scaled_dot_product_attention(q[:, vq], k, v, attn_mask=mask[vq])
        (o * torch.tensor(dO[r].transpose(1, 0, 2))[:, vq]).sum().backward()
        s = (q[:, vq] @ k.transpose(1, 2)) / math.sqrt(dh)
        lse = torch.logsumexp(s.masked_fill(~mask[vq], -math.inf), dim=-1)
        out["O"][r][vq.numpy()] = o.detach().numpy().transpose(1, 0, 2)
        out["lse"][r][vq.numpy()] = lse.detach().numpy().T
        out["dQ"][r] = q.grad.numpy().transpose(1, 0, 2)
        out["dKt"][r] = kt.grad.numpy().transpose(1, 0, 2)
        out["dVt"][r] = vt.grad.numpy().transpose(1, 0, 2)
        out["dKp"][p0:p1] = kp.grad.numpy().transpose(1, 0, 2)
        out["dVp"][p0:p1] = vp.grad.numpy().transpose(1, 0, 2)
    return out


@pytest.mark.parametrize("name", ["ta_tiny", "ta_small"])
def test_tree_attention_matches_torch_sdpa_autograd(name):
    inp, a, dO = _inputs(name)
    if name == "ta_small":                     # keep the CPU suite fast: three requests
        inp = tracegen.gen_tree_attn(name, requests=[0, 1, 2])
        a, dO = TA.from_inputs(inp), TA.bf16_bits_to_f64(inp["dO_bits"])
    O, lse = TA.tree_attention_fwd(**a)
    g = TA.tree_attention_bwd(dO=dO, **a)
    ref = _torch_ref(a, dO)
    np.testing.assert_allclose(O, ref["O"], rtol=1e-10, atol=1e-12)
    fin = np.isfinite(ref["lse"])
    assert np.array_equal(fin, np.isfinite(lse))
    np.testing.assert_allclose(lse[fin], ref["lse"][fin], rtol=1e-12)
    for k, got in zip(["dQ", "dKt", "dVt", "dKp", "dVp"], g):
        np.testing.assert_allclose(got, ref[k], rtol=1e-9, atol=1e-12, err_msg=k)


def test_chain_without_prefix_is_causal_attention():
    rng = np.random.default_rng(5)
    R, N, Hq, Hkv, dh = 2, 7, 4, 4, 16
    Q = rng.standard_normal((R, N + 1, Hq, dh))
    Kt = rng.standard_normal((R, N + 1, Hkv, dh))
    Vt = rng.standard_normal((R, N + 1, Hkv, dh))
    Kp = np.zeros((0, Hkv, dh))
    O, _ = TA.tree_attention_fwd(Q, Kt, Vt, Kp, Kp, np.zeros(R + 1, np.int64))
    for r in range(R):
        o = F.scaled_dot_product_attention(torch.tensor(Q[r].transpose(1, 0, 2)), torch.tensor(Kt[r].transpose(1, 0, 2)),
                                           torch.tensor(Vt[r].transpose(1, 0, 2)), is_causal=True)
        np.testing.assert_allclose(O[r], o.numpy().transpose(1, 0, 2), rtol=1e-12, atol=1e-13)


def test_bruteforce_scalar_loops():
    inp, a, dO = _inputs("ta_tiny")
    O, lse = TA.tree_attention_fwd(**a)
    R, N1, Hq, dh = a["Q"].shape
    G = Hq // a["Kt"].shape[2]
    scale = 1.0 / math.sqrt(dh)
    off = a["prefix_off"]
    for r in range(R):
        par = a["parents"][r]
        for s in range(N1):
            # keys: walk up from node s-1 with plain pointer chasing, written out again here
            tree_keys = {0, s}
            n = s - 1
            while n >= 0:
                tree_keys.add(n + 1)
                n = int(par[n])
            for h in range(Hq):
                keys, vals = [], []
                for j in range(int(off[r]), int(off[r + 1])):
                    keys.append(a["Kp"][j, h // G])
                    vals.append(a["Vp"][j, h // G])
                for t in sorted(tree_keys):
                    keys.append(a["Kt"][r, t, h // G])
                    vals.append(a["Vt"][r, t, h // G])
                sc = [sum(a["Q"][r, s, h, i] * k[i] for i in range(dh)) * scale for k in keys]
                mx = max(sc)
                den = sum(math.exp(x - mx) for x in sc)
                for i in range(dh):
                    num = sum(math.exp(x - mx) * v[i] for x, v in zip(sc, vals))
                    assert abs(O[r, s, h, i] - num / den) < 1e-12
                assert abs(lse[r, s, h] - (mx + math.log(den))) < 1e-12


def test_finite_differences():
    inp, a, dO = _inputs("ta_tiny")
    g = dict(zip(["Q", "Kt", "Vt", "Kp", "Vp"], TA.tree_attention_bwd(dO=dO, **a)))
    rng = np.random.default_rng(11)
    eps = 1e-6

    def f(b):
        O, _ = TA.tree_attention_fwd(**b)
        return float(np.sum(O * dO))

    for name in ["Q", "Kt", "Vt", "Kp", "Vp"]:
        for _ in range(4):
            idx = tuple(int(rng.integers(0, s)) for s in a[name].shape)
            b = dict(a)
            x = a[name].copy()
            x[idx] += eps
            b[name] = x
            fp = f(b)
            x[idx] -= 2 * eps
            fm = f(b)
            fd = (fp - fm) / (2 * eps)
            assert abs(fd - g[name][idx]) <= 1e-6 * max(1.0, abs(fd)), (name, idx, fd, g[name][idx])


def test_branch_independence():
    """Perturbing the K/V of a tree row changes exactly the rows it is an ancestor-or-self
    of (the sibling branches are invisible: P:163-169)."""
    inp, a, dO = _inputs("ta_tiny")
    O0, _ = TA.tree_attention_fwd(**a)
    par = a["parents"]
    N = a["Q"].shape[1] - 1
    for r in range(a["Q"].shape[0]):
        for t in range(1, N + 1):
            b = dict(a)
            Kt = a["Kt"].copy()
            Kt[r, t] += 1.0
            b["Kt"] = Kt
            O1, _ = TA.tree_attention_fwd(**b)
            for s in range(N + 1):
                n, anc = s - 1, {s}
                while n >= 0:
                    anc.add(n + 1)
                    n = int(par[r, n])
                changed = not np.allclose(O1[r, s], O0[r, s], rtol=0, atol=0)
                assert changed == (t in anc), (r, s, t)
            others = [q for q in range(a["Q"].shape[0]) if q != r]
            assert np.array_equal(O1[others], O0[others])


def test_single_key_identity_and_padding():
    rng = np.random.default_rng(3)
    Q = rng.standard_normal((1, 3, 2, 4))
    Kt = rng.standard_normal((1, 3, 1, 4))
    Vt = rng.standard_normal((1, 3, 1, 4))
    empty = np.zeros((0, 1, 4))
    O, lse = TA.tree_attention_fwd(Q, Kt, Vt, empty, empty, np.array([0, 0]), parents=np.array([[-1, 0]]),
                                   num_nodes=np.array([0]))
    # the root sees only itself: softmax of one score is 1
    np.testing.assert_allclose(O[0, 0], np.repeat(Vt[0, 0], 2, axis=0), rtol=0, atol=1e-15)
    np.testing.assert_allclose(lse[0, 0], Q[0, 0] @ Kt[0, 0, 0] / 2.0, rtol=1e-14)
    # padded nodes: zero output, lse -inf, zero gradients
    assert np.all(O[0, 1:] == 0) and np.all(np.isneginf(lse[0, 1:]))
    g = TA.tree_attention_bwd(Q, Kt, Vt, empty, empty, np.array([0, 0]), np.ones_like(Q),
                              parents=np.array([[-1, 0]]), num_nodes=np.array([0]))
    assert np.all(g[0][0, 1:] == 0) and np.all(g[1][0, 1:] == 0) and np.all(g[2][0, 1:] == 0)


def test_gqa_equals_repeated_kv():
    inp, a, dO = _inputs("ta_tiny")
    G = a["Q"].shape[2] // a["Kt"].shape[2]
    O, lse = TA.tree_attention_fwd(**a)
    g = TA.tree_attention_bwd(dO=dO, **a)
    b = dict(a)
    for k in ["Kt", "Vt", "Kp", "Vp"]:
        b[k] = np.repeat(a[k], G, axis=-2)
    O2, lse2 = TA.tree_attention_fwd(**b)
    g2 = TA.tree_attention_bwd(dO=dO, **b)
    np.testing.assert_allclose(O2, O, rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(g2[0], g[0], rtol=1e-12, atol=1e-14)
    # the G repeated copies' gradients sum to the shared head's gradient
    for i, k in [(1, "Kt"), (2, "Vt"), (3, "Kp"), (4, "Vp")]:
        summed = g2[i].reshape(g2[i].shape[:-2] + (-1, G, g2[i].shape[-1])).sum(axis=-2)
        np.testing.assert_allclose(summed, g[i], rtol=1e-12, atol=1e-13, err_msg=k)


def test_sample_subset_is_exact():
    """gen_tree_attn(requests=...) reproduces those requests; the oracle on the subset
    equals the full run on those rows (requests are independent)."""
    full = TA.fwd_bwd(tracegen.gen_tree_attn("ta_tiny"))
    sub = TA.fwd_bwd(tracegen.gen_tree_attn("ta_tiny", requests=[2, 0]))
    np.testing.assert_array_equal(sub["O"], full["O"][[2, 0]])
    np.testing.assert_array_equal(sub["dQ"], full["dQ"][[2, 0]])


# ---------------------------------------------------------------- F4-R6 tree positions + RoPE
def test_tree_positions_are_prefix_plus_depth():
    par = np.array([-1, -1, 0, 0, 1, 3], dtype=np.int32)     # depths 1 1 2 2 2 3
    pos = TA.tree_positions(par, 6, 6, 100)
    assert pos.tolist() == [100, 101, 101, 102, 102, 102, 103]
    assert TA.tree_positions(None, 4, 4, 7).tolist() == [7, 8, 9, 10, 11]     # chain = causal positions
    assert TA.tree_positions(par, 2, 6, 0).tolist() == [0, 1, 1, -1, -1, -1, -1]  # padded nodes


def test_rope_matches_transformers_llama_rotary():
    """Pinned to the library routine the targets use (transformers' apply_rotary_pos_emb with
    Llama's inv_freq = theta^(-2i/dh) and cos/sin of pos * inv_freq repeated over both halves)."""
    from transformers.models.llama.modeling_llama import apply_rotary_pos_emb
    rng = np.random.default_rng(2)
    rows, H, dh, theta = 9, 3, 16, 500000.0
    q = rng.standard_normal((rows, H, dh))
    k = rng.standard_normal((rows, 1, dh))
    pos = np.array([5, 6, 6, 7, 7, 7, 2040, 0, 1])
    inv = 1.0 / (theta ** (torch.arange(0, dh, 2, dtype=torch.float64) / dh))
    fr = torch.tensor(pos, dtype=torch.float64)[:, None] * inv[None, :]
    emb = torch.cat([fr, fr], dim=-1)
    qt, kt = apply_rotary_pos_emb(torch.tensor(q).transpose(0, 1)[None], torch.tensor(k).transpose(0, 1)[None],
                                  emb.cos()[None], emb.sin()[None])
    np.testing.assert_allclose(TA.rope(q, pos, theta), qt[0].transpose(0, 1).numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(TA.rope(k, pos, theta), kt[0].transpose(0, 1).numpy(), rtol=1e-12, atol=1e-12)


def test_rope_invariants():
    rng = np.random.default_rng(4)
    x = rng.standard_normal((6, 2, 32))
    pos = np.array([0, 3, 3, 9, -1, 2047])
    y = TA.rope(x, pos, 10000.0)
    np.testing.assert_allclose(np.linalg.norm(y, axis=-1), np.linalg.norm(x, axis=-1), rtol=1e-13)   # rotation
    np.testing.assert_allclose(TA.rope(y, pos, 10000.0, inverse=True), x, rtol=1e-12, atol=1e-12)    # inverse
    assert np.array_equal(y[4], x[4])                                                                 # pos < 0
    # relative positions: <R(m) q, R(n) k> depends only on m - n
    q, k = rng.standard_normal((1, 1, 32)), rng.standard_normal((1, 1, 32))
    dot = lambda m, n: float(np.sum(TA.rope(q, np.array([m]), 1e4) * TA.rope(k, np.array([n]), 1e4)))
    assert abs(dot(10, 7) - dot(103, 100)) < 1e-10 and abs(dot(0, 0) - float(np.sum(q * k))) < 1e-12

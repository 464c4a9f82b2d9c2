"""Pins for the F4 draft-layer oracle (oracle/draft_layer.py, reading F4-R7) against things
other than itself (-m "not gpu"): torch float64 autograd of an independently written torch
module (F.silu, torch.rsqrt norms, transformers' apply_rotary_pos_emb, scaled_dot_product_attention
with a mask built from boolean matrix powers) for H and every gradient, and central finite
differences through the whole layer."""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import draft_layer as DL
from oracle import tree_attention as TA


def _case(seed=0):
    rng = np.random.default_rng(seed)
    R, N, d, Hq, Hkv, dh, I = 2, 4, 16, 4, 2, 8, 24
    parents = np.array([[-1, -1, 0, 1], [-1, 0, 1, 1]], dtype=np.int32)
    num_nodes = np.array([4, 3], dtype=np.int32)
    lens = [3, 0]
    off = np.array([0, 3, 3])
    n = lambda *s, sc=1.0: rng.standard_normal(s) * sc
    P = dict(Wfc=n(d, 3 * d, sc=0.2), we=1 + n(d, sc=0.1), wh=1 + n(d, sc=0.1), Wq=n(Hq * dh, 2 * d, sc=0.2),
             Wk=n(Hkv * dh, 2 * d, sc=0.2), Wv=n(Hkv * dh, 2 * d, sc=0.2), Wo=n(d, Hq * dh, sc=0.2),
             wpost=1 + n(d, sc=0.1), wfinal=1 + n(d, sc=0.1), Wg=n(I, d, sc=0.2), Wu=n(I, d, sc=0.2), Wd=n(d, I, sc=0.2))
    X = dict(h3=n(R, N + 1, 3 * d), e=n(R, N + 1, d), Kp=n(sum(lens), Hkv, dh), Vp=n(sum(lens), Hkv, dh),
             prefix_off=off, parents=parents, num_nodes=num_nodes)
    cfg = dict(Hq=Hq, Hkv=Hkv, dh=dh, theta=10000.0, eps=1e-6)
    dH = n(R, N + 1, d)
    return P, X, cfg, dH


def _torch_layer(P, X, cfg):
    """Independent torch f64 implementation; returns H and the leaf tensors."""
    T = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in P.items()}
    for k in ("h3", "e", "Kp", "Vp"):
        T[k] = torch.tensor(X[k], dtype=torch.float64, requires_grad=True)
    from transformers.models.llama.modeling_llama import apply_rotary_pos_emb
    R, N1 = X["h3"].shape[:2]
    N = N1 - 1
    Hq, Hkv, dh, eps = cfg["Hq"], cfg["Hkv"], cfg["dh"], cfg["eps"]
    G = Hq // Hkv
    rms = lambda x, w: x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w
    g = T["h3"] @ T["Wfc"].T
    u = torch.cat([rms(T["e"], T["we"]), rms(g, T["wh"])], dim=-1)
    q = (u @ T["Wq"].T).view(R, N1, Hq, dh)
    k = (u @ T["Wk"].T).view(R, N1, Hkv, dh)
    v = (u @ T["Wv"].T).view(R, N1, Hkv, dh)
    inv = 1.0 / (cfg["theta"] ** (torch.arange(0, dh, 2, dtype=torch.float64) / dh))
    outs = []
    off = X["prefix_off"]
    for r in range(R):
        nn = int(X["num_nodes"][r])
        Pr = int(off[r + 1] - off[r])
        # positions: depth by repeated parent lookups (written independently of the oracle's walk)
        depth = [0] * N1
        valid = [True] + [n < nn for n in range(N)]
        for n in range(nn):
            dd, p = 1, int(X["parents"][r][n])
            while p >= 0:
                dd, p = dd + 1, int(X["parents"][r][p])
            depth[n + 1] = dd
        pos = torch.tensor([Pr + dd for dd in depth], dtype=torch.float64)
        emb = torch.cat([pos[:, None] * inv[None, :]] * 2, dim=-1)
        qr, kr = apply_rotary_pos_emb(q[r].transpose(0, 1)[None], k[r].transpose(0, 1)[None], emb.cos()[None],
                                      emb.sin()[None])
        vmask = torch.tensor(valid)
        # keep padded rows unrotated (the oracle leaves them as they are)
        qr = torch.where(vmask[None, None, :, None], qr, q[r].transpose(0, 1)[None])
        kr = torch.where(vmask[None, None, :, None], kr, k[r].transpose(0, 1)[None])
        A = torch.zeros(N1, N1, dtype=torch.float64)
        for n in range(nn):
            A[n + 1, int(X["parents"][r][n]) + 1] = 1.0
        C = torch.eye(N1, dtype=torch.float64)
        for _ in range(N1):
            C = (C @ (torch.eye(N1, dtype=torch.float64) + A)).clamp(max=1.0)
        tm = (C > 0) & vmask[:, None] & vmask[None, :]
        mask = torch.cat([vmask[:, None].expand(N1, Pr), tm], dim=1)
        kk = torch.cat([T["Kp"][off[r]:off[r + 1]].transpose(0, 1), kr[0]], dim=1).repeat_interleave(G, dim=0)
        vv = torch.cat([T["Vp"][off[r]:off[r + 1]].transpose(0, 1), v[r].transpose(0, 1)], dim=1).repeat_interleave(G, dim=0)
        vi = vmask.nonzero().flatten()
        ov = F.scaled_dot_product_attention(qr[0][:, vi], kk, vv, attn_mask=mask[vi])   # [Hq, valid, dh]
        sel = torch.zeros(N1, len(vi), dtype=torch.float64)
        sel[vi, torch.arange(len(vi))] = 1.0                                             # padded rows -> 0
        o = torch.einsum("nv,hvd->nhd", sel, ov)
        outs.append(o.reshape(N1, Hq * dh))
    of = torch.stack(outs)
    y = g + of @ T["Wo"].T
    z = rms(y, T["wpost"])
    h = y + (F.silu(z @ T["Wg"].T) * (z @ T["Wu"].T)) @ T["Wd"].T
    return rms(h, T["wfinal"]), T


def test_draft_layer_matches_torch_autograd():
    P, X, cfg, dH = _case()
    H, S = DL.layer_fwd(P, X, cfg)
    G = DL.layer_bwd(P, X, cfg, S, dH)
    Ht, T = _torch_layer(P, X, cfg)
    np.testing.assert_allclose(H, Ht.detach().numpy(), rtol=1e-10, atol=1e-11)
    (Ht * torch.tensor(dH)).sum().backward()
    for k in list(P) + ["h3", "e", "Kp", "Vp"]:
        np.testing.assert_allclose(G[k], T[k].grad.numpy(), rtol=1e-8, atol=1e-10, err_msg=k)


def test_draft_layer_finite_differences():
    P, X, cfg, dH = _case(3)
    H, S = DL.layer_fwd(P, X, cfg)
    G = DL.layer_bwd(P, X, cfg, S, dH)
    rng = np.random.default_rng(9)
    eps = 1e-6
    for name, src in [("Wfc", P), ("Wq", P), ("Wk", P), ("Wd", P), ("wh", P), ("wpost", P), ("wfinal", P), ("h3", X),
                      ("Kp", X)]:
        for _ in range(3):
            idx = tuple(int(rng.integers(0, s)) for s in src[name].shape)
            vals = []
            for sgn in (1, -1):
                src2 = dict(src)
                x = src[name].copy()
                x[idx] += sgn * eps
                src2[name] = x
                Pp, Xp = (src2, X) if src is P else (P, src2)
                vals.append(float(np.sum(DL.layer_fwd(Pp, Xp, cfg)[0] * dH)))
            fd = (vals[0] - vals[1]) / (2 * eps)
            assert abs(fd - G[name][idx]) <= 2e-6 * max(1.0, abs(fd)), (name, idx, fd, G[name][idx])

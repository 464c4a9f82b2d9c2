"""CPU oracle for NEXT row F4, the whole EAGLE-3 draft layer around the tree attention —
TEST INFRASTRUCTURE ONLY (only tests/, smoke() and bench.py's cpu_baseline may import it).

SURVEY §8(f) F4: "The EAGLE-3 fc (3d -> d) plus one decoder layer with the ancestor-closure mask,
fwd and bwd.  It produces H and consumes dH."  The paper ("hidden states are also sent",
P:163-169 tree attention, P:376 D_RPC h_t) does not spell the layer out; reading F4-R7
 follows the EAGLE-3 draft layer of the Llama/Qwen3 speculators:

    g   = h3 Wfc^T                                     fc: concat(low, mid, high) 3d -> d
    u   = [rms(e) * w_e ; rms(g) * w_h]                2d: token embedding | fused hidden
    q,k,v = u Wq^T, u Wk^T, u Wv^T                     GQA heads (Hq, Hkv, dh)
    q,k = RoPE(q, k) at tree positions (F4-R6)
    o   = TreeAttention(q, [Kp; k], [Vp; v])           (oracle/tree_attention.py)
    y   = g + o Wo^T                                   residual on the fused hidden
    z   = rms(y) * w_post
    h   = y + ((silu(z Wg^T) * (z Wu^T)) Wd^T)        SwiGLU MLP, residual
    H   = rms(h) * w_final                             EAGLE-3's final norm before the lm_head
with rms(x) = x / sqrt(mean(x^2) + eps).  H feeds the lm_head path.  Backward: the gradients of <dH, H> for every weight, for h3, e and the
cached prefix K/V — written out step by step (chain rule per op, in reverse order).
Pins: tests/test_draft_layer_oracle.py (torch f64 autograd of an independent torch module,
central finite differences).  Everything float64.
"""
from __future__ import annotations

import numpy as np

from . import tree_attention as TA


def rms_fwd(x, w, eps):
    r = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return x * r * w, r


def rms_bwd(x, w, r, dy):
    """y = x r w, r = (mean(x^2) + eps)^-1/2:  dx = r (w dy) - x r^3 mean(x w dy);  dw = sum(dy x r)."""
    n = x.shape[-1]
    g = dy * w
    dx = r * g - x * (r ** 3) * np.sum(x * g, axis=-1, keepdims=True) / n
    dw = np.sum(dy * x * r, axis=tuple(range(dy.ndim - 1)))
    return dx, dw


def silu(x):
    return x / (1.0 + np.exp(-x))


def layer_fwd(P: dict, X: dict, cfg: dict):
    """P: weights (Wfc [d,3d], we [d], wh [d], Wq [Hq*dh, 2d], Wk, Wv [Hkv*dh, 2d], Wo [d, Hq*dh],
    wpost [d], Wg, Wu [I, d], Wd [d, I], wfinal [d]); X: h3 [R, N+1, 3d], e [R, N+1, d], Kp/Vp, prefix_off,
    parents, num_nodes; cfg: Hq, Hkv, dh, theta, eps.  Returns H and the saved activations."""
    R, N1, _ = X["h3"].shape
    Hq, Hkv, dh = cfg["Hq"], cfg["Hkv"], cfg["dh"]
    eps = cfg["eps"]
    g = X["h3"] @ P["Wfc"].T
    ue, re = rms_fwd(X["e"], P["we"], eps)
    uh, rh = rms_fwd(g, P["wh"], eps)
    u = np.concatenate([ue, uh], axis=-1)
    q = (u @ P["Wq"].T).reshape(R, N1, Hq, dh)
    k = (u @ P["Wk"].T).reshape(R, N1, Hkv, dh)
    v = (u @ P["Wv"].T).reshape(R, N1, Hkv, dh)
    pos = TA.tree_rope_positions(X["prefix_off"], X["parents"], X["num_nodes"], R, N1 - 1)
    qr, kr = TA.rope(q, pos, cfg["theta"]), TA.rope(k, pos, cfg["theta"])
    o, lse = TA.tree_attention_fwd(qr, kr, v, X["Kp"], X["Vp"], X["prefix_off"], X["parents"], X["num_nodes"])
    of = o.reshape(R, N1, Hq * dh)
    y = g + of @ P["Wo"].T
    z, rp = rms_fwd(y, P["wpost"], eps)
    a, b = z @ P["Wg"].T, z @ P["Wu"].T
    m = silu(a) * b
    h = y + m @ P["Wd"].T
    H, rf = rms_fwd(h, P["wfinal"], eps)
    S = dict(g=g, re=re, rh=rh, u=u, pos=pos, qr=qr, kr=kr, v=v, of=of, y=y, z=z, rp=rp, a=a, b=b, m=m, h=h, rf=rf)
    return H, S


def layer_bwd(P: dict, X: dict, cfg: dict, S: dict, dH):
    """Gradients of <dH, H> (reverse order of layer_fwd)."""
    R, N1, _ = X["h3"].shape
    Hq, Hkv, dh = cfg["Hq"], cfg["Hkv"], cfg["dh"]
    G = {}
    flat = lambda t: t.reshape(-1, t.shape[-1])
    # H = rms(h) w_final
    dhid, G["wfinal"] = rms_bwd(S["h"], P["wfinal"], S["rf"], dH)
    # h = y + m Wd^T
    G["Wd"] = flat(dhid).T @ flat(S["m"])
    dm = dhid @ P["Wd"]
    sa = 1.0 / (1.0 + np.exp(-S["a"]))
    da = dm * S["b"] * (sa * (1.0 + S["a"] * (1.0 - sa)))        # d silu(a)/da = s (1 + a (1 - s))
    db = dm * silu(S["a"])
    G["Wg"] = flat(da).T @ flat(S["z"])
    G["Wu"] = flat(db).T @ flat(S["z"])
    dz = da @ P["Wg"] + db @ P["Wu"]
    dy_mlp, G["wpost"] = rms_bwd(S["y"], P["wpost"], S["rp"], dz)
    dy = dhid + dy_mlp
    # y = g + of Wo^T
    G["Wo"] = flat(dy).T @ flat(S["of"])
    do = (dy @ P["Wo"]).reshape(R, N1, Hq, dh)
    dqr, dkr, dv, dKp, dVp = TA.tree_attention_bwd(S["qr"], S["kr"], S["v"], X["Kp"], X["Vp"], X["prefix_off"], do,
                                                   X["parents"], X["num_nodes"])
    G["Kp"], G["Vp"] = dKp, dVp
    dq = TA.rope(dqr, S["pos"], cfg["theta"], inverse=True).reshape(R, N1, Hq * dh)
    dk = TA.rope(dkr, S["pos"], cfg["theta"], inverse=True).reshape(R, N1, Hkv * dh)
    dv = dv.reshape(R, N1, Hkv * dh)
    G["Wq"] = flat(dq).T @ flat(S["u"])
    G["Wk"] = flat(dk).T @ flat(S["u"])
    G["Wv"] = flat(dv).T @ flat(S["u"])
    du = dq @ P["Wq"] + dk @ P["Wk"] + dv @ P["Wv"]
    d = X["e"].shape[-1]
    de, G["we"] = rms_bwd(X["e"], P["we"], S["re"], du[..., :d])
    dg_norm, G["wh"] = rms_bwd(S["g"], P["wh"], S["rh"], du[..., d:])
    dg = dy + dg_norm
    G["Wfc"] = flat(dg).T @ flat(X["h3"])
    G["h3"] = dg @ P["Wfc"]
    G["e"] = de
    return G

"""GPU parity of the F4 draft layer (aurora_draft_layer_fwd/bwd, reading F4-R7) against the f64
oracle (oracle/draft_layer.py, pinned to torch autograd in tests/test_draft_layer_oracle.py) on
identical seeded bf16 inputs.  Tolerances: H at 1e-2 relative Frobenius error (bf16 activations
between the GEMMs), every gradient at the north star's 2e-2."""
import numpy as np
import pytest
import torch

import tracegen
from oracle import draft_layer as DL
from oracle import tree_attention as TA

pytestmark = pytest.mark.gpu


def _bf_round(x):
    return TA.bf16_bits_to_f64(tracegen.f32_to_bf16_bits(np.asarray(x, np.float32)))


def _case(seed=7, chain=False):
    """tree: 3 requests (a beam tree, a chain written as a tree, a ragged tree), one empty prefix;
    chain=True: parents NULL (chain), GQA group 4, one request with no valid node."""
    rng = np.random.default_rng(seed)
    R, N, d, I, Hq, Hkv, dh = 3, 8, 256, 384, 4, 2, 128
    parents = np.array([[-1, -1, 0, 0, 1, 2, 3, 4], [-1, 0, 1, 2, 3, 4, 5, 6], [-1, -1, -1, 0, 1, 2, 3, 3]],
                       dtype=np.int32)
    num_nodes = np.array([8, 8, 6], dtype=np.int32)
    lens = np.array([40, 0, 75])
    if chain:
        R, N, Hq, Hkv = 4, 5, 8, 2
        parents, num_nodes, lens = None, np.array([5, 0, 3, 5], dtype=np.int32), np.array([10, 130, 0, 64])
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    sc = lambda fan: 1.0 / np.sqrt(fan)
    n = lambda *s, k=1.0: rng.standard_normal(s) * k
    P = dict(Wfc=_bf_round(n(d, 3 * d, k=sc(3 * d))), we=1 + n(d, k=0.1), wh=1 + n(d, k=0.1),
             Wq=_bf_round(n(Hq * dh, 2 * d, k=sc(2 * d))), Wk=_bf_round(n(Hkv * dh, 2 * d, k=sc(2 * d))),
             Wv=_bf_round(n(Hkv * dh, 2 * d, k=sc(2 * d))), Wo=_bf_round(n(d, Hq * dh, k=sc(Hq * dh))),
             wpost=1 + n(d, k=0.1), wfinal=1 + n(d, k=0.1), Wg=_bf_round(n(I, d, k=sc(d))), Wu=_bf_round(n(I, d, k=sc(d))),
             Wd=_bf_round(n(d, I, k=sc(I))))
    for k in ("we", "wh", "wpost", "wfinal"):
        P[k] = P[k].astype(np.float32).astype(np.float64)
    X = dict(h3=_bf_round(n(R, N + 1, 3 * d)), e=_bf_round(n(R, N + 1, d)), Kp=_bf_round(n(int(lens.sum()), Hkv, dh)),
             Vp=_bf_round(n(int(lens.sum()), Hkv, dh)), prefix_off=off, parents=parents, num_nodes=num_nodes)
    cfg = dict(Hq=Hq, Hkv=Hkv, dh=dh, theta=500000.0, eps=1e-6, d=d, I=I, R=R, N=N)
    dH = n(R, N + 1, d, k=0.1).astype(np.float32).astype(np.float64)
    return P, X, cfg, dH


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _run_layer(P, X, cfg, dH, reps=1):
    from paper_2602_06932_b200 import aurora as A
    dev = "cuda"
    bf = lambda x: torch.tensor(np.asarray(x, np.float32)).to(torch.bfloat16).to(dev).contiguous()
    f32 = lambda x: torch.tensor(np.asarray(x, np.float32)).to(dev).contiguous()
    W = {k: (f32(v) if k in ("we", "wh", "wpost", "wfinal") else bf(v)) for k, v in P.items()}
    R, N, d, I = cfg["R"], cfg["N"], cfg["d"], cfg["I"]
    M = R * (N + 1)
    poff = torch.tensor(X["prefix_off"], dtype=torch.int32, device=dev)
    par = None if X["parents"] is None else torch.tensor(X["parents"], device=dev)
    ta = A.TreeAttention(R, N, cfg["Hq"], cfg["Hkv"], cfg["dh"], poff, int(np.diff(X["prefix_off"]).max()),
                         parents=par, num_nodes=torch.tensor(X["num_nodes"], device=dev))
    layer = A.DraftLayer(ta, d, I, W, theta=cfg["theta"], eps=cfg["eps"])
    h3, e = bf(X["h3"].reshape(M, 3 * d)), bf(X["e"].reshape(M, d))
    Kp, Vp = bf(X["Kp"]), bf(X["Vp"])
    outs = []
    for _ in range(reps):
        H = torch.empty(M, d, dtype=torch.bfloat16, device=dev)
        layer.forward(h3, e, Kp, Vp, H)
        G = {k: torch.empty(v.shape, dtype=torch.float32, device=dev) for k, v in W.items()}
        dh3 = torch.empty(M, 3 * d, dtype=torch.float32, device=dev)
        de = torch.empty(M, d, dtype=torch.float32, device=dev)
        dKp, dVp = torch.empty_like(Kp), torch.empty_like(Vp)
        layer.backward(h3, e, Kp, Vp, f32(dH.reshape(M, d)), G, dh3, de, dKp, dVp)
        torch.cuda.synchronize()
        assert int(ta.status.item()) == 0
        outs.append(dict(H=H, dh3=dh3, de=de, dKp=dKp, dVp=dVp, **{"G" + k: v for k, v in G.items()}))
    return outs


@pytest.mark.parametrize("chain", [False, True], ids=["tree", "chain_ragged"])
def test_draft_layer_parity(chain):
    P, X, cfg, dH = _case(chain=chain)
    o = _run_layer(P, X, cfg, dH)[0]
    H, dh3, de, dKp, dVp = o["H"], o["dh3"], o["de"], o["dKp"], o["dVp"]
    G = {k: o["G" + k] for k in P}
    Hr, S = DL.layer_fwd(P, X, cfg)
    Gr = DL.layer_bwd(P, X, cfg, S, dH)
    assert _rel(H.float().cpu().numpy().reshape(Hr.shape), Hr) <= 1e-2
    got = {k: G[k].cpu().numpy() for k in G}
    got.update(h3=dh3.cpu().numpy().reshape(Gr["h3"].shape), e=de.cpu().numpy().reshape(Gr["e"].shape),
               Kp=dKp.float().cpu().numpy(), Vp=dVp.float().cpu().numpy())
    errs = {k: _rel(got[k], Gr[k]) for k in Gr}
    print("draft layer rel. Frobenius errors: H %.2e, " % _rel(H.float().cpu().numpy().reshape(Hr.shape), Hr) +
          ", ".join(f"{k} {v:.2e}" for k, v in sorted(errs.items())))
    bad = {k: v for k, v in errs.items() if v > 2e-2}
    assert not bad, errs


def test_draft_layer_deterministic():
    P, X, cfg, dH = _case(seed=11)
    a, b = _run_layer(P, X, cfg, dH, reps=2)
    for k in a:
        assert torch.equal(a[k], b[k]), k


def test_whole_speculator_step_parity():
    """Verification + draft layer + lm_head loss fwd/bwd + draft layer bwd in one step
    (SpeculatorStep) against the oracle chain (draft-layer oracle -> H in f64 -> the lm_head /
    Eq. 3 oracle -> dH -> draft-layer oracle bwd) on the small tree trace."""
    import oracle
    from paper_2602_06932_b200 import aurora as A
    tr = tracegen.gen_trace("small_tree")
    c = tr["cfg"]
    R, N, d, V = c.R, c.N, c.d, c.V
    M = R * (N + 1)
    rng = np.random.default_rng(21)
    I, Hq, Hkv, dh = 256, 2, 1, 128
    lens = rng.integers(0, 80, size=R)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    sc = lambda fan: 1.0 / np.sqrt(fan)
    n = lambda *s, k=1.0: rng.standard_normal(s) * k
    P = dict(Wfc=_bf_round(n(d, 3 * d, k=sc(3 * d))), we=np.ones(d), wh=np.ones(d),
             Wq=_bf_round(n(Hq * dh, 2 * d, k=sc(2 * d))), Wk=_bf_round(n(Hkv * dh, 2 * d, k=sc(2 * d))),
             Wv=_bf_round(n(Hkv * dh, 2 * d, k=sc(2 * d))), Wo=_bf_round(n(d, Hq * dh, k=sc(Hq * dh))),
             wpost=np.ones(d), wfinal=np.ones(d), Wg=_bf_round(n(I, d, k=sc(d))), Wu=_bf_round(n(I, d, k=sc(d))),
             Wd=_bf_round(n(d, I, k=sc(I))))
    X = dict(h3=_bf_round(n(R, N + 1, 3 * d)), e=_bf_round(n(R, N + 1, d)), Kp=_bf_round(n(int(lens.sum()), Hkv, dh)),
             Vp=_bf_round(n(int(lens.sum()), Hkv, dh)), prefix_off=off, parents=tr["parents"], num_nodes=tr["num_nodes"])
    cfg = dict(Hq=Hq, Hkv=Hkv, dh=dh, theta=1000000.0, eps=1e-6)
    # ---- oracle chain
    Hr, S = DL.layer_fwd(P, X, cfg)
    T64 = oracle.bf16_bits_to_f64(tr["T_bits"])
    amax, topk, _ = oracle.target_scan(T64, 10)
    lab = oracle.verify(tr["draft_tokens"], tr["parents"], tr["num_nodes"], amax, 0)
    tg = oracle.row_targets(lab["row_class"], lambda m: T64[m], topk, 1, 10, 1.0, 0)
    fw = oracle.loss_fwd(Hr.reshape(M, d), tr["W_bits"], tg)
    bw = oracle.loss_bwd(Hr.reshape(M, d), tr["W_bits"], tg, fw["lse"])
    Gr = DL.layer_bwd(P, X, cfg, S, bw["dH"].reshape(R, N + 1, d))
    # ---- GPU step
    dev = "cuda"
    bf = lambda x: torch.tensor(np.asarray(x, np.float32)).to(torch.bfloat16).to(dev).contiguous()
    f32 = lambda x: torch.tensor(np.asarray(x, np.float32)).to(dev).contiguous()
    bits = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).to(dev)
    W = {k: (f32(v) if k in ("we", "wh", "wpost", "wfinal") else bf(v)) for k, v in P.items()}
    par = torch.from_numpy(tr["parents"]).to(dev)
    ta = A.TreeAttention(R, N, Hq, Hkv, dh, torch.tensor(off, dtype=torch.int32, device=dev), int(lens.max()),
                         parents=par)
    layer = A.DraftLayer(ta, d, I, W, theta=cfg["theta"], eps=cfg["eps"])
    spec = A.SpecTrainStep(R, N, d, V)
    step = A.SpeculatorStep(spec, layer)
    h3, e, Kp, Vp = bf(X["h3"].reshape(M, 3 * d)), bf(X["e"].reshape(M, d)), bf(X["Kp"]), bf(X["Vp"])
    W_lm = bits(tr["W_bits"])
    H = torch.empty(M, d, dtype=torch.bfloat16, device=dev)
    dH = torch.empty(M, d, dtype=torch.float32, device=dev)
    dW_lm = torch.empty(V, d, dtype=torch.float32, device=dev)
    G = {k: torch.empty(v.shape, dtype=torch.float32, device=dev) for k, v in W.items()}
    dh3 = torch.empty(M, 3 * d, dtype=torch.float32, device=dev)
    de = torch.empty(M, d, dtype=torch.float32, device=dev)
    dKp, dVp = torch.empty_like(Kp), torch.empty_like(Vp)
    loss = step.step(torch.from_numpy(tr["draft_tokens"]).to(dev), bits(tr["T_bits"]), h3, e, Kp, Vp, W_lm, H, dH,
                     dW_lm, G, dh3, de, dKp, dVp, parents=par)
    torch.cuda.synchronize()
    assert int(spec.status.item()) == 0 and int(ta.status.item()) == 0
    assert np.array_equal(spec.accept_len.cpu().numpy(), lab["accept_len"])
    # the layer's H (bf16) against the oracle's f64 H, then the loss at the 1e-3 bar against the
    # oracle evaluated on the H the GPU layer produced (the lm_head stage's own inputs); the chain
    # loss against the all-f64 oracle differs by the bf16 rounding of H
    H_gpu = oracle.bf16_bits_to_f64(H.view(torch.int16).cpu().numpy().view(np.uint16))
    assert _rel(H_gpu, Hr.reshape(M, d)) <= 2e-2
    fw_h = oracle.loss_fwd(H_gpu, tr["W_bits"], tg)
    assert abs(float(loss.item()) - fw_h["loss"]) <= 1e-3 * abs(fw_h["loss"])
    assert abs(float(loss.item()) - fw["loss"]) <= 5e-3 * abs(fw["loss"])
    assert _rel(dW_lm.cpu().numpy(), bw["dW"]) <= 2e-2
    assert _rel(dH.cpu().numpy(), bw["dH"]) <= 2e-2
    got = {k: G[k].cpu().numpy() for k in G}
    got.update(h3=dh3.cpu().numpy().reshape(Gr["h3"].shape), e=de.cpu().numpy().reshape(Gr["e"].shape),
               Kp=dKp.float().cpu().numpy(), Vp=dVp.float().cpu().numpy())
    errs = {k: _rel(got[k], Gr[k]) for k in Gr}
    print("whole step: loss %.6f (oracle %.6f); " % (float(loss.item()), fw["loss"]) +
          ", ".join(f"{k} {v:.2e}" for k, v in sorted(errs.items())))
    assert not {k: v for k, v in errs.items() if v > 2e-2}, errs


def test_whole_step_with_adamw_over_all_params():
    """F3 over the whole speculator: lm_head + draft-layer parameters in one flat master
    (SpeculatorParams), one AdamW step with one global norm after SpeculatorStep.  (1) The flat
    gradient against the oracle chain's, per parameter within 2e-2 relative Frobenius error and the
    global norm within 1e-2; (2) the optimizer arithmetic: the GPU update equals oracle.adamw_step
    applied to the GPU's own gradient buffer (fp32 vs f64, rtol 2e-6)."""
    import oracle
    from paper_2602_06932_b200 import aurora as A
    tr = tracegen.gen_trace("small_tree")
    c = tr["cfg"]
    R, N, d, V = c.R, c.N, c.d, c.V
    M = R * (N + 1)
    rng = np.random.default_rng(31)
    I, Hq, Hkv, dh = 256, 2, 1, 128
    lens = rng.integers(0, 80, size=R)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    sc = lambda fan: 1.0 / np.sqrt(fan)
    n = lambda *s, k=1.0: rng.standard_normal(s) * k
    P = dict(Wfc=_bf_round(n(d, 3 * d, k=sc(3 * d))), we=np.ones(d), wh=np.ones(d),
             Wq=_bf_round(n(Hq * dh, 2 * d, k=sc(2 * d))), Wk=_bf_round(n(Hkv * dh, 2 * d, k=sc(2 * d))),
             Wv=_bf_round(n(Hkv * dh, 2 * d, k=sc(2 * d))), Wo=_bf_round(n(d, Hq * dh, k=sc(Hq * dh))),
             wpost=np.ones(d), wfinal=np.ones(d), Wg=_bf_round(n(I, d, k=sc(d))), Wu=_bf_round(n(I, d, k=sc(d))),
             Wd=_bf_round(n(d, I, k=sc(I))))
    X = dict(h3=_bf_round(n(R, N + 1, 3 * d)), e=_bf_round(n(R, N + 1, d)), Kp=_bf_round(n(int(lens.sum()), Hkv, dh)),
             Vp=_bf_round(n(int(lens.sum()), Hkv, dh)), prefix_off=off, parents=tr["parents"], num_nodes=tr["num_nodes"])
    cfg = dict(Hq=Hq, Hkv=Hkv, dh=dh, theta=1000000.0, eps=1e-6)
    W_lm64 = TA.bf16_bits_to_f64(tr["W_bits"])
    # ---- oracle chain + oracle AdamW over the flat parameter vector (same order as SpeculatorParams)
    Hr, S = DL.layer_fwd(P, X, cfg)
    T64 = oracle.bf16_bits_to_f64(tr["T_bits"])
    amax, topk, _ = oracle.target_scan(T64, 10)
    lab = oracle.verify(tr["draft_tokens"], tr["parents"], tr["num_nodes"], amax, 0)
    tg = oracle.row_targets(lab["row_class"], lambda m: T64[m], topk, 1, 10, 1.0, 0)
    fw = oracle.loss_fwd(Hr.reshape(M, d), tr["W_bits"], tg)
    bw = oracle.loss_bwd(Hr.reshape(M, d), tr["W_bits"], tg, fw["lse"])
    Gr = DL.layer_bwd(P, X, cfg, S, bw["dH"].reshape(R, N + 1, d))
    order = ["Wfc", "Wq", "Wk", "Wv", "Wo", "Wg", "Wu", "Wd", "we", "wh", "wpost", "wfinal"]
    w0 = np.concatenate([W_lm64.ravel()] + [np.asarray(P[k], np.float32).astype(np.float64).ravel() for k in order])
    g64 = np.concatenate([bw["dW"].ravel()] + [Gr[k].ravel() for k in order])
    lr = 1e-3
    w1, _, _, norm = oracle.adamw_step(w0, np.zeros_like(w0), np.zeros_like(w0), g64, 1, lr, warmup_steps=0)
    # ---- GPU: flat parameters, whole step, one AdamW step
    dev = "cuda"
    sp = A.SpeculatorParams(d, I, Hq, Hkv, dh, V, dev)
    sp.load(dict(W_lm=W_lm64, **{k: P[k] for k in order}))
    par = torch.from_numpy(tr["parents"]).to(dev)
    ta = A.TreeAttention(R, N, Hq, Hkv, dh, torch.tensor(off, dtype=torch.int32, device=dev), int(lens.max()),
                         parents=par)
    layer = A.DraftLayer(ta, d, I, sp.W, theta=cfg["theta"], eps=cfg["eps"])
    step = A.SpeculatorStep(A.SpecTrainStep(R, N, d, V), layer)
    bf = lambda x: torch.tensor(np.asarray(x, np.float32)).to(torch.bfloat16).to(dev).contiguous()
    bits = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).to(dev)
    h3, e, Kp, Vp = bf(X["h3"].reshape(M, 3 * d)), bf(X["e"].reshape(M, d)), bf(X["Kp"]), bf(X["Vp"])
    H = torch.empty(M, d, dtype=torch.bfloat16, device=dev)
    dH = torch.empty(M, d, dtype=torch.float32, device=dev)
    dh3 = torch.empty(M, 3 * d, dtype=torch.float32, device=dev)
    de = torch.empty(M, d, dtype=torch.float32, device=dev)
    dKp, dVp = torch.empty_like(Kp), torch.empty_like(Vp)
    step.step(torch.from_numpy(tr["draft_tokens"]).to(dev), bits(tr["T_bits"]), h3, e, Kp, Vp, sp.W_lm, H, dH,
              sp.dW_lm, sp.G, dh3, de, dKp, dVp, parents=par)
    torch.cuda.synchronize()
    g_gpu = sp.grad.cpu().numpy().astype(np.float64)
    w_before = sp.master.cpu().numpy().astype(np.float64)
    o = 0
    for name, gref in [("W_lm", bw["dW"])] + [(k, Gr[k]) for k in order]:
        nel = gref.size
        assert _rel(g_gpu[o:o + nel], gref.ravel()) <= 2e-2, name
        o += nel
    opt = sp.adamw(lr=lr, warmup_steps=0)
    sp.optimizer_step(opt)
    torch.cuda.synchronize()
    assert abs(float(opt.grad_norm.item()) - norm) <= 1e-2 * norm
    f32 = lambda x: float(np.float32(x))
    w_ref, _, _, norm_gpu = oracle.adamw_step(w_before, np.zeros_like(w0), np.zeros_like(w0), g_gpu, 1, f32(lr),
                                              beta1=f32(0.9), beta2=f32(0.999), eps=f32(1e-8), warmup_steps=0)
    assert abs(float(opt.grad_norm.item()) - norm_gpu) <= 2e-5 * norm_gpu
    np.testing.assert_allclose(sp.master.cpu().numpy(), w_ref, rtol=2e-6, atol=1e-9)
    # the bf16 copy the GEMMs read was refreshed from the updated master
    np.testing.assert_allclose(sp.bf.float().cpu().numpy(), sp.master.cpu().numpy(), rtol=2 ** -8, atol=1e-30)


def test_speculator_step_rejects_a_different_tree():
    """verification must follow the tree the layer's TreeAttention was built with."""
    from paper_2602_06932_b200 import aurora as A
    dev = "cuda"
    R, N, d, I, Hq, Hkv, dh, V = 2, 4, 256, 256, 2, 1, 128, 1000
    par = torch.tensor([[-1, 0, 1, 2], [-1, 0, 0, 1]], dtype=torch.int32, device=dev)
    off = torch.tensor([0, 5, 9], dtype=torch.int32, device=dev)
    ta = A.TreeAttention(R, N, Hq, Hkv, dh, off, 5, parents=par)
    bf = lambda *s: torch.zeros(*s, dtype=torch.bfloat16, device=dev)
    W = dict(Wfc=bf(d, 3 * d), Wq=bf(Hq * dh, 2 * d), Wk=bf(Hkv * dh, 2 * d), Wv=bf(Hkv * dh, 2 * d), Wo=bf(d, Hq * dh),
             Wg=bf(I, d), Wu=bf(I, d), Wd=bf(d, I), **{k: torch.ones(d, device=dev) for k in ("we", "wh", "wpost", "wfinal")})
    step = A.SpeculatorStep(A.SpecTrainStep(R, N, d, V), A.DraftLayer(ta, d, I, W))
    other = par.clone()
    with pytest.raises(ValueError):
        step.step(None, None, None, None, None, None, None, None, None, None, None, None, None, None, None,
                  parents=other)

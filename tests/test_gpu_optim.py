"""GPU parity of the NEXT F3 optimizer step (aurora_adamw_step) vs the f64 oracle O7.

fp32 arithmetic against f64: the update of one element is a handful of fp32 operations,
so W, m, v agree to a few fp32 ulps; the norm is an fp32 sum of n squares (relative
error ~1e-6 at these sizes).
"""
import numpy as np
import pytest
import torch

import oracle
import tracegen
from paper_2602_06932_b200 import aurora as A

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    A.lib()


def _bf16_rne(x32: np.ndarray) -> np.ndarray:
    return tracegen.f32_to_bf16_bits(x32)


def _f32(x: float) -> float:
    """The C-ABI takes fp32 hyperparameters (0.999f = 0.99900001...); the oracle gets the
    value the library actually received."""
    return float(np.float32(x))


HP = dict(beta1=_f32(0.9), beta2=_f32(0.999), eps=_f32(1e-8))


@pytest.mark.parametrize("n,grad_scale,wd,warmup", [(4 * 100003, 1e-3, 0.0, 400), (4096 * 257, 1e-6, 0.01, 3),
                                                     (1 << 22, 1e-2, 0.0, 0)])
def test_adamw_parity(n, grad_scale, wd, warmup):
    inp = tracegen.gen_adamw_inputs(n, steps=3, grad_scale=grad_scale)
    W = torch.from_numpy(inp["W"].copy()).cuda()
    Wb = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    opt = A.AdamW(W, lr=1e-4, weight_decay=wd, warmup_steps=warmup)
    Wr, mr, vr = inp["W"].astype(np.float64), np.zeros(n), np.zeros(n)
    for step, g in enumerate(inp["G"], start=1):
        opt.step(torch.from_numpy(g).cuda(), W_bf16=Wb)
        Wr, mr, vr, norm = oracle.adamw_step(Wr, mr, vr, g, step, _f32(1e-4), weight_decay=_f32(wd),
                                             max_grad_norm=0.5, warmup_steps=warmup, **HP)
        torch.cuda.synchronize()
        assert abs(float(opt.grad_norm.item()) - norm) <= 2e-5 * norm
        np.testing.assert_allclose(W.cpu().numpy(), Wr, rtol=2e-6, atol=1e-9)
        # m, v: sums of two fp32 terms that can cancel -> a few fp32 ulps of the operand scale
        np.testing.assert_allclose(opt.m.cpu().numpy(), mr, rtol=1e-5, atol=4e-7 * np.abs(mr).max())
        np.testing.assert_allclose(opt.v.cpu().numpy(), vr, rtol=1e-5, atol=4e-7 * np.abs(vr).max())
    # the bf16 copy is the RNE rounding of the fp32 master
    np.testing.assert_array_equal(Wb.view(torch.int16).cpu().numpy().view(np.uint16), _bf16_rne(W.cpu().numpy()))


def test_adamw_extra_sq_and_validation():
    n = 4096
    inp = tracegen.gen_adamw_inputs(n, steps=1, grad_scale=1e-2)
    W = torch.from_numpy(inp["W"].copy()).cuda()
    opt = A.AdamW(W, lr=1e-3, warmup_steps=0)
    extra = torch.tensor([3.0], device="cuda")
    opt.step(torch.from_numpy(inp["G"][0]).cuda(), extra_sq=extra)
    Wr, _, _, norm = oracle.adamw_step(inp["W"], np.zeros(n), np.zeros(n), inp["G"][0], 1, _f32(1e-3), warmup_steps=0,
                                       extra_sq=3.0, **HP)
    torch.cuda.synchronize()
    assert abs(float(opt.grad_norm.item()) - norm) <= 1e-5 * norm
    np.testing.assert_allclose(W.cpu().numpy(), Wr, rtol=2e-6, atol=1e-9)
    with pytest.raises(Exception):  # n % 4 != 0
        A.aurora_adamw_step(W[:4093], None, opt.m[:4093], opt.v[:4093], torch.zeros(4093, device="cuda"), 1, opt.cfg,
                            opt.ws)


def _bf16(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def _prepare(tr):
    c = tr["cfg"]
    H, W = _bf16(tr["H_bits"]), _bf16(tr["W_bits"])
    draft = torch.from_numpy(tr["draft_tokens"]).cuda()
    par = None if tr["parents"] is None else torch.from_numpy(tr["parents"]).cuda()
    nn = None if tr["num_nodes"] is None else torch.from_numpy(tr["num_nodes"]).cuda()
    st = A.SpecTrainStep(c.R, c.N, c.d, c.V)
    st.verify(draft, _bf16(tr["T_bits"]), par, nn)
    return c, H, W, st


@pytest.mark.parametrize("qe", [0, 1, 2])
@pytest.mark.parametrize("name", ["small", "small_tree", "mid"])
def test_fused_bwd_adamw_matches_unfused(name, qe):
    """F3 fused into the dW epilogue (dW never stored) vs bwd + aurora_adamw_step: same dH
    bits, the same update up to the norm's summation order; and the oracle's AdamW applied
    to the unfused dW pins the arithmetic.  Both state-entry shapes of the fused kernel
    (128 x 32 entries shared by all epilogue warps; qe 1 / 2: 32 x 128 / 32 x 64 entries per lane
    quadrant)."""
    saved = A.aurora_get_option("dw_adamw_qe")
    A.aurora_set_option("dw_adamw_qe", qe)
    try:
        _fused_vs_unfused(name)
    finally:
        A.aurora_set_option("dw_adamw_qe", saved)


def _fused_vs_unfused(name):
    tr = tracegen.gen_trace(name)
    c, H, W1, st1 = _prepare(tr)
    st1.forward(H, W1)
    dH1 = torch.empty(c.M, c.d, device="cuda")
    dW1 = torch.empty(c.V, c.d, device="cuda")
    st1.backward(H, W1, dH1, dW1)
    W0 = W1.float().clone()
    opt1 = A.AdamW(W1.float().reshape(-1).clone(), lr=1e-4, warmup_steps=0)
    opt1.step(dW1.reshape(-1), W_bf16=W1.reshape(-1))
    _, _, W2, st2 = _prepare(tr)
    st2.forward(H, W2)
    dH2 = torch.empty(c.M, c.d, device="cuda")
    opt2 = A.AdamW(W2.float().reshape(-1).clone(), lr=1e-4, warmup_steps=0)
    st2.backward_adamw(H, W2, dH2, opt2)
    torch.cuda.synchronize()
    assert torch.equal(dH1, dH2)
    n1, n2 = float(opt1.grad_norm.item()), float(opt2.grad_norm.item())
    # the fused path takes the Gram form of the norm for small M (sum over M^2 products of fp32
    # Gram entries instead of V*d squares): equal up to fp32 summation order, ~1e-5 relative
    assert abs(n1 - n2) <= 1e-4 * n1
    np.testing.assert_allclose(opt2.W.cpu().numpy(), opt1.W.cpu().numpy(), rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(opt2.m.cpu().numpy(), opt1.m.cpu().numpy(), rtol=1e-4,
                               atol=1e-6 * float(opt1.m.abs().max()))
    assert (W2.float() - opt2.W.reshape(c.V, c.d)).abs().max() <= 4e-3 * W0.abs().max()  # bf16 copy of the master
    f32 = lambda x: float(np.float32(x))
    Wr, mr, vr, norm = oracle.adamw_step(W0.reshape(-1).cpu().numpy(), np.zeros(W0.numel()), np.zeros(W0.numel()),
                                         dW1.reshape(-1).cpu().numpy(), 1, f32(1e-4), warmup_steps=0,
                                         beta1=f32(0.9), beta2=f32(0.999), eps=f32(1e-8))
    assert abs(n2 - norm) <= 1e-4 * norm
    np.testing.assert_allclose(opt2.W.cpu().numpy(), Wr, rtol=2e-6, atol=1e-9)


@pytest.mark.parametrize("name", ["small", "mid"])
def test_fused_gram_norm_equals_sum_of_squares(name):
    """The Gram-form norm (||dZ^T H||_F^2 = sum (dZ dZ^T) .* (H H^T)) against the dW-recompute
    sum-of-squares path of the same fused call (option gram_norm)."""
    tr = tracegen.gen_trace(name)
    norms = []
    saved = A.aurora_get_option("gram_norm")
    try:
        for gram in (1, 0):
            A.aurora_set_option("gram_norm", gram)
            c, H, W, st = _prepare(tr)
            st.forward(H, W)
            opt = A.AdamW(W.float().reshape(-1).clone(), lr=1e-4, warmup_steps=0)
            st.backward_adamw(H, W, torch.empty(c.M, c.d, device="cuda"), opt)
            torch.cuda.synchronize()
            norms.append(float(opt.grad_norm.item()))
    finally:
        A.aurora_set_option("gram_norm", saved)
    assert abs(norms[0] - norms[1]) <= 1e-4 * norms[1]


def test_fused_bwd_adamw_needs_one_chunk():
    tr = tracegen.gen_trace("small")
    c, H, W, st = _prepare(tr)
    saved = A.aurora_get_option("dz_chunk_bytes")
    try:
        A.aurora_set_option("dz_chunk_bytes", 64 << 10)
        st = A.SpecTrainStep(c.R, c.N, c.d, c.V)
        st.verify(torch.from_numpy(tr["draft_tokens"]).cuda(), _bf16(tr["T_bits"]), None,
                  torch.from_numpy(tr["num_nodes"]).cuda() if tr["num_nodes"] is not None else None)
        st.forward(H, W)
        opt = A.AdamW(W.float().reshape(-1).clone())
        with pytest.raises(A.AuroraError) as ei:
            st.backward_adamw(H, W, torch.empty(c.M, c.d, device="cuda"), opt)
        assert ei.value.status == 5
    finally:
        A.aurora_set_option("dz_chunk_bytes", saved)


def test_adamw_device_step_counter_graph_replay():
    """The step counter lives on the device: three replays of ONE captured optimizer step
    follow the oracle's steps 1, 2, 3 (warm-up LR and bias corrections advance)."""
    n = 4 * 4099
    inp = tracegen.gen_adamw_inputs(n, steps=1, grad_scale=1e-2)
    W = torch.from_numpy(inp["W"].copy()).cuda()
    g = torch.from_numpy(inp["G"][0]).cuda()
    opt = A.AdamW(W, lr=1e-3, warmup_steps=5)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        opt.step(g)            # eager step 1 (also warms up the launch path)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        opt.step(g)
    Wr, mr, vr = inp["W"].astype(np.float64), np.zeros(n), np.zeros(n)
    Wr, mr, vr, _ = oracle.adamw_step(Wr, mr, vr, inp["G"][0], 1, _f32(1e-3), warmup_steps=5, **HP)
    for step in (2, 3, 4):
        graph.replay()
        torch.cuda.synchronize()
        Wr, mr, vr, _ = oracle.adamw_step(Wr, mr, vr, inp["G"][0], step, _f32(1e-3), warmup_steps=5, **HP)
        np.testing.assert_allclose(W.cpu().numpy(), Wr, rtol=2e-6, atol=1e-9)


def test_extra_sq_added_once_after_vp_allreduce():
    """extra_sq (other parameter groups) enters the global norm once: with a 1-rank comm
    (the VP allreduce runs as an identity) the result equals the comm-less call."""
    n = 4096
    inp = tracegen.gen_adamw_inputs(n, steps=1, grad_scale=1e-2)
    extra = torch.tensor([2.0], device="cuda")
    uid = A.aurora_comm_get_unique_id()
    comm = A.aurora_comm_create(uid, 1, 0, 1, 1)
    try:
        outs = []
        for c in (None, comm):
            W = torch.from_numpy(inp["W"].copy()).cuda()
            opt = A.AdamW(W, lr=1e-3, warmup_steps=0, comm=c)
            opt.step(torch.from_numpy(inp["G"][0]).cuda(), extra_sq=extra)
            torch.cuda.synchronize()
            outs.append((W.cpu().numpy(), float(opt.grad_norm.item())))
        assert outs[0][1] == outs[1][1]
        assert np.array_equal(outs[0][0], outs[1][0])
        _, _, _, norm = oracle.adamw_step(inp["W"], np.zeros(n), np.zeros(n), inp["G"][0], 1, _f32(1e-3),
                                          warmup_steps=0, extra_sq=2.0, **HP)
        assert abs(outs[0][1] - norm) <= 1e-5 * norm
    finally:
        A.aurora_comm_destroy(comm)

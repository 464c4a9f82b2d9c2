"""GPU parity: the CUDA path (through the C-ABI) vs the f64 oracle on identical
seeded traces (-m gpu).  Tolerances (BASELINE.json north_star): labels and
accept lengths bit-exact; loss within 1e-3 relative; dW and dH within 2e-2
relative Frobenius error.
"""
import os

import numpy as np
import pytest
import torch

# every buffer handed to the C-ABI is created with an explicit dtype; guard against a
# process-wide default dtype change by another test module
assert torch.get_default_dtype() == torch.float32

import oracle
import tracegen
from paper_2602_06932_b200 import aurora as A

pytestmark = pytest.mark.gpu

LOSS_RTOL = 1e-3
GRAD_RFRO = 2e-2


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    A.lib()


def _bf16(bits: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def _to_gpu(tr):
    g = dict(T=_bf16(tr["T_bits"]), H=_bf16(tr["H_bits"]), W=_bf16(tr["W_bits"]),
             draft=torch.from_numpy(tr["draft_tokens"]).cuda())
    g["parents"] = None if tr["parents"] is None else torch.from_numpy(tr["parents"]).cuda()
    g["num_nodes"] = None if tr["num_nodes"] is None else torch.from_numpy(tr["num_nodes"]).cuda()
    return g


def _run_gpu(tr, want_grads=True, **kw):
    c = tr["cfg"]
    g = _to_gpu(tr)
    st = A.SpecTrainStep(c.R, c.N, c.d, c.V, **kw)
    st.verify(g["draft"], g["T"], g["parents"], g["num_nodes"])
    st.forward(g["H"], g["W"])
    out = dict(st=st, g=g)
    if want_grads:
        dH = torch.empty(c.M, c.d, dtype=torch.float32, device="cuda")
        dW = torch.empty(c.V, c.d, dtype=torch.float32, device="cuda")
        st.backward(g["H"], g["W"], dH, dW)
        out["dH"], out["dW"] = dH, dW
    torch.cuda.synchronize()
    return out


def _rfro(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _check_labels(st, ref, tr, k_accept=1, k_discard=10, h_rtol=0.0):
    assert int(st.status.item()) == 0
    np.testing.assert_array_equal(st.target_argmax.cpu().numpy(), ref["argmax"])
    np.testing.assert_array_equal(st.accepted.cpu().numpy(), ref["accepted"])
    np.testing.assert_array_equal(st.accept_len.cpu().numpy(), ref["accept_len"])
    np.testing.assert_array_equal(st.bonus.cpu().numpy(), ref["bonus"])
    np.testing.assert_array_equal(st.row_class.cpu().numpy(), ref["row_class"])
    tg = ref["targets"]
    assert tuple(st.counts.cpu().tolist()) == tuple(tg["counts"])
    sup = st.sup_idx.cpu().numpy()
    sp = st.sup_p.cpu().numpy()
    w = st.row_w.cpu().numpy()
    Hh = st.row_H.cpu().numpy()
    for m in range(tr["M"]):
        k = len(tg["sup_idx"][m])
        np.testing.assert_array_equal(sup[m, :k], tg["sup_idx"][m])
        assert (sup[m, k:] == np.iinfo(np.int32).max).all()
        np.testing.assert_allclose(sp[m, :k], tg["sup_p"][m], rtol=2e-6, atol=1e-7)
        assert abs(w[m] - tg["w"][m]) <= 1e-6 * abs(tg["w"][m]) + 1e-12
        assert abs(Hh[m] - tg["H"][m]) <= 1e-5 + h_rtol * abs(tg["H"][m])


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 520, 192), (37, 70, 200), (512, 1024, 1024)])
def test_gemm_engine_vs_torch_fp32(a_mn, b_mn, M, N, K):
    """Test hook: the tcgen05 engine on a plain GEMM vs a PyTorch fp32 reference."""
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    Am = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    Bm = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
    ref = Am.float() @ Bm.float().T
    Ast = Am.T.contiguous() if a_mn else Am
    Bst = Bm.T.contiguous() if b_mn else Bm
    # pad leading dims to 16 B multiples
    def pad(x):
        c = x.shape[1]
        cp = (c + 7) // 8 * 8
        y = torch.zeros(x.shape[0], cp, dtype=x.dtype, device=x.device)
        y[:, :c] = x
        return y
    Ast, Bst = pad(Ast), pad(Bst)
    D = torch.full((M, N), float("nan"), device="cuda", dtype=torch.float32)
    A.aurora_debug_gemm(bool(a_mn), bool(b_mn), Ast, Bst, D, M, N, K, Ast.stride(0), Bst.stride(0), D.stride(0))
    torch.cuda.synchronize()
    err = (D - ref).abs().max().item()
    assert err <= 1e-3 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("name", ["tiny", "small", "small_tree", "mid"])
def test_full_parity_small(name):
    tr = tracegen.gen_trace(name)
    ref = oracle.step(tr)
    out = _run_gpu(tr)
    st = out["st"]
    _check_labels(st, ref, tr)
    loss = float(st.loss.item())
    assert abs(loss - ref["loss"]) <= LOSS_RTOL * abs(ref["loss"]), (loss, ref["loss"])
    np.testing.assert_allclose(st.row_lse.cpu().numpy(), ref["lse"], rtol=2e-5, atol=1e-5)
    assert _rfro(out["dW"].cpu().numpy(), ref["dW"]) <= GRAD_RFRO
    assert _rfro(out["dH"].cpu().numpy(), ref["dH"]) <= GRAD_RFRO


@pytest.mark.parametrize("kw", [dict(k_accept=3, k_discard=16), dict(lambda_discard=0.0), dict(normalize=1),
                                dict(discard_scope=1, lambda_discard=2.5), dict(k_accept=1, k_discard=1)])
def test_loss_config_variants(kw):
    tr = tracegen.gen_trace("small_tree")
    ref = oracle.step(tr, **kw)
    out = _run_gpu(tr, **kw)
    _check_labels(out["st"], ref, tr)
    loss = float(out["st"].loss.item())
    assert abs(loss - ref["loss"]) <= LOSS_RTOL * abs(ref["loss"]) + 1e-9
    assert _rfro(out["dW"].cpu().numpy(), ref["dW"]) <= GRAD_RFRO
    assert _rfro(out["dH"].cpu().numpy(), ref["dH"]) <= GRAD_RFRO


def test_edge_shapes():
    """R=1, N=1, V < one tile, d = 64: single partial tile in every GEMM."""
    for cfg in [tracegen.TraceConfig("e1", d=64, V=100, R=1, N=1, seed=9, alpha=(0.5,)),
                tracegen.TraceConfig("e2", d=128, V=257, R=3, N=32, seed=10, alpha=(0.9,)),
                tracegen.TraceConfig("e3", d=64, V=20, R=70, N=2, seed=11, alpha=(0.5,), ragged=True)]:
        tr = tracegen.gen_trace(cfg)
        ref = oracle.step(tr)
        out = _run_gpu(tr)
        _check_labels(out["st"], ref, tr)
        loss = float(out["st"].loss.item())
        assert abs(loss - ref["loss"]) <= LOSS_RTOL * abs(ref["loss"])
        assert _rfro(out["dW"].cpu().numpy(), ref["dW"]) <= GRAD_RFRO
        assert _rfro(out["dH"].cpu().numpy(), ref["dH"]) <= GRAD_RFRO


def test_all_rejected_and_all_accepted():
    tr = tracegen.gen_trace(tracegen.TraceConfig("rej", d=64, V=500, R=6, N=5, seed=12, alpha=(0.0,)))
    ref = oracle.step(tr)
    out = _run_gpu(tr)
    _check_labels(out["st"], ref, tr)
    assert (ref["accept_len"] == 1).all()
    tr = tracegen.gen_trace(tracegen.TraceConfig("acc", d=64, V=500, R=6, N=5, seed=13, alpha=(1.0,)))
    ref = oracle.step(tr)
    out = _run_gpu(tr)
    _check_labels(out["st"], ref, tr)
    assert (ref["accept_len"] == 6).all() and ref["targets"]["counts"][1] == 0
    assert abs(float(out["st"].loss.item()) - ref["loss"]) <= LOSS_RTOL * abs(ref["loss"])


def test_status_word_errors():
    tr = tracegen.gen_trace("small")
    c = tr["cfg"]
    # non-finite logit
    T = tr["T_bits"].copy()
    T[3, 17] = 0x7FC0  # NaN
    g = _to_gpu(tr)
    st = A.SpecTrainStep(c.R, c.N, c.d, c.V)
    st.verify(g["draft"], _bf16(T), g["parents"], g["num_nodes"])
    torch.cuda.synchronize()
    assert int(st.status.item()) & A.STATUS_NONFINITE
    # out-of-range token
    d2 = g["draft"].clone()
    d2[0, 0] = c.V
    st.verify(d2, g["T"], g["parents"], g["num_nodes"])
    torch.cuda.synchronize()
    assert int(st.status.item()) & A.STATUS_RANGE
    # malformed parents
    p = torch.full((c.R, c.N), -1, dtype=torch.int32, device="cuda")
    p[0, 2] = 2
    st.verify(g["draft"], g["T"], p, g["num_nodes"])
    torch.cuda.synchronize()
    assert int(st.status.item()) & A.STATUS_STRUCTURE
    # clean again
    st.verify(g["draft"], g["T"], g["parents"], g["num_nodes"])
    torch.cuda.synchronize()
    assert int(st.status.item()) == 0


def test_dlogits_rows_hook_and_row_sum_zero():
    tr = tracegen.gen_trace("small")
    ref = oracle.step(tr)
    out = _run_gpu(tr)
    rows = [0, 5, 11, tr["M"] - 1]
    dz = out["st"].debug_dlogits_rows(out["g"]["H"], out["g"]["W"], rows).cpu().numpy().astype(np.float64)
    H64 = oracle.bf16_bits_to_f64(tr["H_bits"])
    dz_ref = oracle.dlogits_rows(H64, tr["W_bits"], ref["targets"], ref["lse"][rows], rows)
    for i in range(len(rows)):
        assert _rfro(dz[i], dz_ref[i]) <= 1e-3 or np.abs(dz_ref[i]).max() == 0
    assert np.abs(dz.sum(1)).max() <= 1e-5 * max(1e-30, np.abs(dz).max()) * tr["V"] ** 0.5 + 1e-7
    # dW column sums vanish (row-sum-zero of dZ)
    dW = out["dW"].cpu().numpy().astype(np.float64)
    assert np.abs(dW.sum(0)).max() <= 2e-2 * np.abs(dW).sum(0).max()


def test_accumulate_and_upstream_grad():
    tr = tracegen.gen_trace("small")
    out = _run_gpu(tr)
    st, g = out["st"], out["g"]
    c = tr["cfg"]
    dH2 = torch.empty_like(out["dH"])
    dW2 = out["dW"].clone()
    dl = torch.tensor([-2.0], device="cuda", dtype=torch.float32)
    st.forward(g["H"], g["W"])   # re-stage the numerators (the first backward consumed them)
    st.backward(g["H"], g["W"], dH2, dW2, dloss=dl, accumulate_dW=True)
    torch.cuda.synchronize()
    # dW2 = dW + (-2) dW = -dW ; dH2 = -2 dH
    assert _rfro(dW2.cpu().numpy(), -out["dW"].cpu().numpy()) < 1e-5
    assert _rfro(dH2.cpu().numpy(), -2 * out["dH"].cpu().numpy()) < 1e-5


def test_determinism():
    tr = tracegen.gen_trace("mid")
    a = _run_gpu(tr)
    b = _run_gpu(tr)
    assert a["st"].loss.item() == b["st"].loss.item()
    assert torch.equal(a["dW"], b["dW"]) and torch.equal(a["dH"], b["dH"])


def test_llama_full_size_parity():
    """configs[1] at full size, in the launch configuration bench.py times:
    labels bit-exact on all rows, loss / dW / dH against the full f64 oracle."""
    tr = tracegen.gen_trace("llama")
    out = _run_gpu(tr)
    ref = oracle.step(tr)
    _check_labels(out["st"], ref, tr)
    loss = float(out["st"].loss.item())
    assert abs(loss - ref["loss"]) <= LOSS_RTOL * abs(ref["loss"])
    assert _rfro(out["dW"].cpu().numpy(), ref["dW"]) <= GRAD_RFRO
    assert _rfro(out["dH"].cpu().numpy(), ref["dH"]) <= GRAD_RFRO


@pytest.mark.parametrize("name", ["qwen3", "minimax", "tree"])
def test_large_config_sampled_parity(name):
    """Full-size configs: labels bit-exact on every row (oracle scan row by row),
    per-row lse / loss on sampled rows, dW column-sum property at full size."""
    tr = tracegen.gen_trace(name)
    out = _run_gpu(tr, want_grads=True)
    st = out["st"]
    M, V = tr["M"], tr["V"]
    T = tr["T_bits"]
    am = np.empty(M, dtype=np.int64)
    topk = np.empty((M, 10), dtype=np.int64)
    for m0 in range(0, M, 256):
        a, t, nf = oracle.target_scan(oracle.bf16_bits_to_f64(T[m0:m0 + 256]), 10)
        assert not nf
        am[m0:m0 + 256], topk[m0:m0 + 256] = a, t
    lab = oracle.verify(tr["draft_tokens"], tr["parents"], tr["num_nodes"], am)
    np.testing.assert_array_equal(st.target_argmax.cpu().numpy(), am)
    np.testing.assert_array_equal(st.accept_len.cpu().numpy(), lab["accept_len"])
    np.testing.assert_array_equal(st.row_class.cpu().numpy(), lab["row_class"])
    np.testing.assert_array_equal(st.bonus.cpu().numpy(), lab["bonus"])
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(M, size=24, replace=False))
    tg = oracle.row_targets(lab["row_class"], lambda m: oracle.bf16_bits_to_f64(T[m]), topk, rows=rows)
    H64 = oracle.bf16_bits_to_f64(tr["H_bits"])
    fw = oracle.loss_fwd(H64, tr["W_bits"], tg, rows=rows)
    np.testing.assert_allclose(st.row_lse.cpu().numpy()[rows], fw["lse"], rtol=2e-5)
    np.testing.assert_allclose(st.row_loss.cpu().numpy()[rows], fw["row_loss"], rtol=1e-3, atol=1e-3)
    dW = out["dW"].double()
    colsum = dW.sum(0).abs().max().item()
    assert colsum <= 2e-2 * dW.abs().sum(0).max().item()


def test_single_rank_comm_runs_every_exchange_identically():
    """A 1-rank NCCL communicator runs C1-C5 as identity collectives: results must be
    bit-identical to the comm-less path (exercises dlopen'd NCCL, CommSplit, AllGather,
    AllReduce on the caller's stream)."""
    tr = tracegen.gen_trace("small_tree")
    base = _run_gpu(tr)
    uid = A.aurora_comm_get_unique_id()
    comm = A.aurora_comm_create(uid, 1, 0, 1, 1)
    try:
        out = _run_gpu(tr, comm=comm)
        for k in ("target_argmax", "accept_len", "row_class", "sup_idx", "sup_p", "row_w", "row_lse", "loss"):
            assert torch.equal(getattr(out["st"], k), getattr(base["st"], k)), k
        assert torch.equal(out["dW"], base["dW"]) and torch.equal(out["dH"], base["dH"])
    finally:
        A.aurora_comm_destroy(comm)


@pytest.mark.parametrize("cuts", [(2600,), (1000, 2049, 4100)])
def test_emulated_vocab_parallel_shards(cuts):
    """VP shard maths on one GPU through the C-ABI: global labels, then per-shard fwd
    with vocab_offset (support entries outside the shard, shard sizes not multiples of
    256), host combine of the per-shard (lse, u) exactly as C3 does, per-shard bwd with
    the global lse, dW shards concatenated and dH summed (C4)."""
    tr = tracegen.gen_trace("small")
    ref = oracle.step(tr)
    c = tr["cfg"]
    full = _run_gpu(tr, want_grads=False)
    st, g = full["st"], full["g"]
    bounds = [0, *cuts, c.V]
    lses, us = [], []
    M = c.M
    for v0, v1 in zip(bounds[:-1], bounds[1:]):
        Ws = g["W"][v0:v1].contiguous()
        row_lse = torch.empty(M, device="cuda", dtype=torch.float32)
        row_loss = torch.empty(M, device="cuda", dtype=torch.float32)
        loss = torch.empty(1, device="cuda", dtype=torch.float32)
        A.aurora_spec_loss_fwd(g["H"], Ws, M, c.d, v1 - v0, v0, st.labels, row_lse, row_loss, loss,
                               st.ws.data_ptr(), st.ws_bytes)
        torch.cuda.synchronize()
        lses.append(row_lse.double())
        us.append(row_lse.double() + st.row_H.double() - row_loss.double())   # u_p = lse_p + H~ - l_p
    L = torch.stack(lses)
    lse = torch.logsumexp(L, 0)
    pad = st.row_class == A.ROW_PAD
    row_loss = torch.where(pad, torch.zeros_like(lse), lse - torch.stack(us).sum(0) + st.row_H.double())
    loss = float((st.row_w.double() * row_loss).sum())
    assert abs(loss - ref["loss"]) <= 1e-3 * abs(ref["loss"])
    np.testing.assert_allclose(lse.cpu().numpy(), ref["lse"], rtol=2e-5)
    glse = lse.float().contiguous()
    dH = torch.zeros(M, c.d, device="cuda", dtype=torch.float64)  # host-side accumulation only
    dWs = []
    for v0, v1 in zip(bounds[:-1], bounds[1:]):
        Ws = g["W"][v0:v1].contiguous()
        dHp = torch.empty(M, c.d, device="cuda", dtype=torch.float32)
        dWp = torch.empty(v1 - v0, c.d, device="cuda", dtype=torch.float32)
        A.aurora_spec_loss_bwd(g["H"], Ws, M, c.d, v1 - v0, v0, st.labels, glse, None, dHp, dWp, False, False,
                               st.ws.data_ptr(), st.ws_bytes)
        torch.cuda.synchronize()
        dH += dHp.double()
        dWs.append(dWp)
    dW = torch.cat(dWs, 0)
    assert _rfro(dW.cpu().numpy(), ref["dW"]) <= GRAD_RFRO
    assert _rfro(dH.cpu().numpy(), ref["dH"]) <= GRAD_RFRO


@pytest.fixture
def option():
    """Set library execution options for one test, restoring them afterwards."""
    saved = {}

    def set_(name, value):
        if name not in saved:
            saved[name] = A.aurora_get_option(name)
        A.aurora_set_option(name, value)

    yield set_
    for k, v in saved.items():
        A.aurora_set_option(k, v)


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(256, 256, 64), (300, 520, 192), (37, 70, 200), (1024, 512, 1024)])
def test_gemm_engine_cta_pair(option, a_mn, b_mn, M, N, K):
    """tcgen05.mma.cta_group::2 (2-CTA cluster, M=256 pair tiles) vs PyTorch fp32."""
    option("gemm_pair", 2)
    test_gemm_engine_vs_torch_fp32(a_mn, b_mn, M, N, K)


@pytest.mark.parametrize("pair", [1, 2])
@pytest.mark.parametrize("name", ["tiny", "small_tree", "mid"])
def test_parity_forced_tiling(option, name, pair):
    option("gemm_pair", pair)
    test_full_parity_small(name)


@pytest.mark.parametrize("tile_n", [224, 192])
@pytest.mark.parametrize("name", ["tiny", "small_tree", "mid"])
def test_parity_narrow_tiles(option, name, tile_n):
    """fwd / dz GEMMs with 224- and 192-column vocab tiles (single-CTA tiles)."""
    option("gemm_pair", 1)
    option("tile_n", tile_n)
    test_full_parity_small(name)


def test_narrow_tiles_emulated_vp(option):
    """Ragged vocab shards (tails not multiples of 224 / 192) with narrow tiles."""
    option("gemm_pair", 1)
    for t in (224, 192):
        option("tile_n", t)
        test_emulated_vocab_parallel_shards((1000, 2049, 4100))


@pytest.mark.parametrize("name", ["tiny", "small", "small_tree", "mid"])
def test_parity_fused_bwd(option, name):
    """The whole backward as one persistent kernel (unified DZ/DH/DW tile queue)."""
    option("bwd_mode", 1)
    test_full_parity_small(name)


def test_fused_bwd_emulated_vp_and_serial(option):
    option("bwd_mode", 1)
    test_emulated_vocab_parallel_shards((1000, 2049, 4100))
    option("bwd_mode", 0)
    option("bwd_concurrent", 1)   # dW || dH on the library's side streams
    test_full_parity_small("small")
    test_determinism()


def _run_gpu_topk(tr, **kw):
    c = tr["cfg"]
    g = _to_gpu_base(tr)
    ids = torch.from_numpy(tr["Tk_idx"]).cuda()
    vals = torch.from_numpy(np.ascontiguousarray(tr["Tk_bits"]).view(np.int16)).view(torch.bfloat16).cuda()
    st = A.SpecTrainStep(c.R, c.N, c.d, c.V, **kw)
    st.verify_topk(g["draft"], ids, vals, g["parents"], g["num_nodes"])
    st.forward(g["H"], g["W"])
    dH = torch.empty(c.M, c.d, dtype=torch.float32, device="cuda")
    dW = torch.empty(c.V, c.d, dtype=torch.float32, device="cuda")
    st.backward(g["H"], g["W"], dH, dW)
    torch.cuda.synchronize()
    return st, dH, dW


def _to_gpu_base(tr):
    g = dict(H=_bf16(tr["H_bits"]), W=_bf16(tr["W_bits"]), draft=torch.from_numpy(tr["draft_tokens"]).cuda())
    g["parents"] = None if tr["parents"] is None else torch.from_numpy(tr["parents"]).cuda()
    g["num_nodes"] = None if tr["num_nodes"] is None else torch.from_numpy(tr["num_nodes"]).cuda()
    return g


@pytest.mark.parametrize("name,K_t", [("tiny", 64), ("small", 1024), ("small_tree", 100), ("mid", 1024)])
def test_topk_ingest_parity(name, K_t):
    """NEXT F1: labels from the transmitted top-K payload bit-exact vs the oracle's sparse
    scan; loss / dW / dH within the north-star tolerances."""
    tr = tracegen.gen_trace_topk(name, K_t=K_t)
    ref = oracle.step_topk(tr)
    st, dH, dW = _run_gpu_topk(tr)
    _check_labels(st, ref, tr)
    loss = float(st.loss.item())
    assert abs(loss - ref["loss"]) <= LOSS_RTOL * abs(ref["loss"])
    assert _rfro(dW.cpu().numpy(), ref["dW"]) <= GRAD_RFRO
    assert _rfro(dH.cpu().numpy(), ref["dH"]) <= GRAD_RFRO


def test_topk_ingest_matches_dense_path():
    """The dense path and the sparse path give identical labels when the payload holds
    every column of the dense rows (a shuffled full row)."""
    tr = tracegen.gen_trace("small")
    c = tr["cfg"]
    rng = np.random.default_rng(3)
    perm = np.stack([rng.permutation(c.V) for _ in range(c.M)]).astype(np.int32)
    tr["Tk_idx"] = perm
    tr["Tk_bits"] = np.take_along_axis(tr["T_bits"], perm, 1)
    dense = _run_gpu(tr)
    st, dH, dW = _run_gpu_topk(tr)
    for k in ("target_argmax", "accepted", "accept_len", "bonus", "row_class", "sup_idx", "counts"):
        assert torch.equal(getattr(st, k), getattr(dense["st"], k)), k
    assert torch.allclose(st.sup_p, dense["st"].sup_p)
    assert torch.equal(dW, dense["dW"]) and torch.equal(dH, dense["dH"])


def test_topk_ingest_status_bits():
    tr = tracegen.gen_trace_topk("small", K_t=64)
    c = tr["cfg"]
    g = _to_gpu_base(tr)
    ids = torch.from_numpy(tr["Tk_idx"]).cuda()
    vals = torch.from_numpy(np.ascontiguousarray(tr["Tk_bits"]).view(np.int16)).view(torch.bfloat16).cuda()
    st = A.SpecTrainStep(c.R, c.N, c.d, c.V)
    bad = ids.clone()
    bad[2, 5] = c.V + 3
    st.verify_topk(g["draft"], bad, vals, g["parents"], g["num_nodes"])
    torch.cuda.synchronize()
    assert int(st.status.item()) & A.STATUS_RANGE
    v2 = vals.clone()
    v2[4, 0] = float("inf")
    st.verify_topk(g["draft"], ids, v2, g["parents"], g["num_nodes"])
    torch.cuda.synchronize()
    assert int(st.status.item()) & A.STATUS_NONFINITE


@pytest.mark.parametrize("name,K_t,ka,kd", [("tiny", 64, 64, 64), ("small", 256, 200, 17), ("small_tree", 100, 32, 100),
                                           ("mid", 1024, 1024, 1024)])
def test_topk_long_support_parity(name, K_t, ka, kd):
    """F1 soft distillation: supports of up to 1024 transmitted pairs per row (CTA-per-row
    bitonic sort + long finalize; binary-search seek in the GEMM epilogues).  H~ sums
    up to 1024 fp32 terms, hence a relative allowance on it."""
    tr = tracegen.gen_trace_topk(name, K_t=K_t)
    ref = oracle.step_topk(tr, k_accept=ka, k_discard=kd)
    st, dH, dW = _run_gpu_topk(tr, k_accept=ka, k_discard=kd)
    _check_labels(st, ref, tr, h_rtol=2e-6)
    loss = float(st.loss.item())
    assert abs(loss - ref["loss"]) <= LOSS_RTOL * abs(ref["loss"])
    assert _rfro(dW.cpu().numpy(), ref["dW"]) <= GRAD_RFRO
    assert _rfro(dH.cpu().numpy(), ref["dH"]) <= GRAD_RFRO


def test_topk_long_support_status_and_limits():
    tr = tracegen.gen_trace_topk("small", K_t=64)
    c = tr["cfg"]
    g = _to_gpu_base(tr)
    ids = torch.from_numpy(tr["Tk_idx"]).cuda()
    vals = torch.from_numpy(np.ascontiguousarray(tr["Tk_bits"]).view(np.int16)).view(torch.bfloat16).cuda()
    st = A.SpecTrainStep(c.R, c.N, c.d, c.V, k_accept=40, k_discard=40)
    dup = ids.clone()
    dup[3, :2] = dup[3, 0]             # the same id twice among the row's pairs, both in the top
    vd = vals.clone()
    vd[3, :2] = 60.0
    st.verify_topk(g["draft"], dup, vd, g["parents"], g["num_nodes"])
    torch.cuda.synchronize()
    assert int(st.status.item()) & A.STATUS_STRUCTURE
    bad = ids.clone()
    bad[2, 5] = -1
    st.verify_topk(g["draft"], bad, vals, g["parents"], g["num_nodes"])
    torch.cuda.synchronize()
    assert int(st.status.item()) & A.STATUS_RANGE
    with pytest.raises(Exception):     # k above the transmitted K_t
        A.SpecTrainStep(c.R, c.N, c.d, c.V, k_accept=65).verify_topk(g["draft"], ids, vals, g["parents"],
                                                                      g["num_nodes"])
    with pytest.raises(Exception):     # dense verify keeps k <= 16
        big = A.SpecTrainStep(c.R, c.N, c.d, c.V, k_accept=17)
        T = torch.zeros(c.M, c.V, dtype=torch.bfloat16, device="cuda")
        big.verify(g["draft"], T, g["parents"], g["num_nodes"])


# ----------------------------------------------------------------------------- F2 objectives
F2_VARIANTS = [dict(accept_loss="rkl", ntp_beta=0.0, k_discard=10), dict(accept_loss="rkl", ntp_beta=0.5, k_discard=0),
               dict(accept_loss="fkl", ntp_beta=0.0, k_discard=0), dict(accept_loss="rkl", ntp_beta=1.0, k_discard=3)]


def _check_f2(name, kw, **run_kw):
    tr = tracegen.gen_trace(name)
    ref = oracle.step_variants(tr, **kw)
    out = _run_gpu(tr, **kw, **run_kw)
    st = out["st"]
    assert int(st.status.item()) == 0
    np.testing.assert_array_equal(st.target_argmax.cpu().numpy(), ref["argmax"])
    np.testing.assert_array_equal(st.accept_len.cpu().numpy(), ref["accept_len"])
    np.testing.assert_array_equal(st.row_class.cpu().numpy(), ref["row_class"])
    assert tuple(st.counts.cpu().tolist()) == tuple(ref["counts"])
    valid = ref["row_class"] != oracle.PAD
    np.testing.assert_allclose(st.row_loss.cpu().numpy()[valid], ref["row_loss"][valid], rtol=1e-3, atol=2e-4)
    loss = float(st.loss.item())
    assert abs(loss - ref["loss"]) <= LOSS_RTOL * abs(ref["loss"]), (loss, ref["loss"])
    assert _rfro(out["dW"].cpu().numpy(), ref["dW"]) <= GRAD_RFRO
    assert _rfro(out["dH"].cpu().numpy(), ref["dH"]) <= GRAD_RFRO


@pytest.mark.parametrize("kw", F2_VARIANTS)
@pytest.mark.parametrize("name", ["tiny", "small", "small_tree", "mid"])
def test_f2_objectives_parity(name, kw):
    """NEXT F2 (§5.1 objectives): reverse KL on ACCEPT rows (+NTP), dense KL(p || q) on
    DISCARD rows ("top-k = 0"), vs the oracle's direct full-row definitions."""
    _check_f2(name, kw)


@pytest.mark.parametrize("opt", [dict(gemm_pair=2), dict(gemm_pair=1, tile_n=224), dict(bwd_mode=1)])
def test_f2_objectives_other_launch_configs(option, opt):
    """CTA pairs, narrow tiles, and bwd_mode=1 (routed to the chunked path for F2)."""
    for k, v in opt.items():
        option(k, v)
    _check_f2("mid", F2_VARIANTS[1])
    _check_f2("small_tree", F2_VARIANTS[3])


@pytest.mark.parametrize("budget", [64 << 10, 700 << 10])
@pytest.mark.parametrize("name", ["small", "small_tree", "mid"])
def test_parity_multi_chunk_bwd(option, name, budget):
    """A small dz_chunk_bytes budget splits the backward into several dZ^T vocab chunks
    (the default keeps the whole local vocabulary in one): dH accumulates over chunks,
    each dW chunk lands at its own rows."""
    option("dz_chunk_bytes", budget)
    test_full_parity_small(name)
    _check_f2(name, F2_VARIANTS[1])


@pytest.mark.parametrize("name", ["small", "small_tree", "mid"])
def test_dw_resident_matches_streamed(option, name):
    """A8 for K = M <= 512: the A-resident CTA-pair sweep (opt-in) issues the same MMA
    sequence per tile as the streamed pair kernel, so dW is bit-identical; both match the
    oracle."""
    tr = tracegen.gen_trace(name)
    option("dw_resident", 1)
    a = _run_gpu(tr)
    option("dw_resident", 0)
    b = _run_gpu(tr)
    assert torch.equal(a["dW"], b["dW"]) and torch.equal(a["dH"], b["dH"])
    ref = oracle.step(tr)
    assert _rfro(a["dW"].cpu().numpy(), ref["dW"]) <= GRAD_RFRO


def test_single_rank_comm_f2_objectives():
    """F2 under a (1-rank) vocab-parallel communicator: the T row statistics go through the
    VP triple allgather + ordered merge, (m, s, u, r) through C3; results match the
    comm-less path (the merge of one triple reproduces it up to the log/exp round trip)
    and the oracle."""
    tr = tracegen.gen_trace("small")
    kw = F2_VARIANTS[1]
    base = _run_gpu(tr, **kw)
    ref = oracle.step_variants(tr, **kw)
    uid = A.aurora_comm_get_unique_id()
    comm = A.aurora_comm_create(uid, 1, 0, 1, 1)
    try:
        out = _run_gpu(tr, comm=comm, **kw)
        for k in ("target_argmax", "accept_len", "row_class", "sup_idx", "row_w"):
            assert torch.equal(getattr(out["st"], k), getattr(base["st"], k)), k
        np.testing.assert_allclose(out["st"].row_lse_t.cpu().numpy(), base["st"].row_lse_t.cpu().numpy(), rtol=1e-6)
        loss = float(out["st"].loss.item())
        assert abs(loss - ref["loss"]) <= LOSS_RTOL * abs(ref["loss"])
        assert _rfro(out["dW"].cpu().numpy(), ref["dW"]) <= GRAD_RFRO
        assert _rfro(out["dH"].cpu().numpy(), ref["dH"]) <= GRAD_RFRO
    finally:
        A.aurora_comm_destroy(comm)


@pytest.mark.parametrize("name", ["tiny", "small", "small_tree", "mid"])
def test_parity_recompute_bwd(option, name):
    """fwd_stage = 0: the round-1 backward that recomputes Z tiles in a dz GEMM (the
    default stages exp(z - m_half) in the forward and rescales it); both match the oracle."""
    option("fwd_stage", 0)
    test_full_parity_small(name)


def test_staged_and_recompute_backward_agree(option):
    """The staged backward (no recompute GEMM) and the recompute backward give the same
    gradients up to bf16 rounding of dz (one extra rounding of the staged numerators)."""
    tr = tracegen.gen_trace("mid")
    a = _run_gpu(tr)
    option("fwd_stage", 0)
    b = _run_gpu(tr)
    # the staged fwd takes an exact per-(row, tile half) max before the exp sums, the
    # recompute path an online one: same loss up to fp32 summation order
    assert abs(float(a["st"].loss.item()) - float(b["st"].loss.item())) <= 1e-6 * abs(float(b["st"].loss.item()))
    assert _rfro(a["dW"].cpu().numpy(), b["dW"].cpu().numpy()) <= 5e-3
    assert _rfro(a["dH"].cpu().numpy(), b["dH"].cpu().numpy()) <= 5e-3


def test_staged_record_consumed_and_invalidated():
    """A second backward after one forward, or a verify between forward and backward,
    falls back to the recompute path (the staged numerators are consumed / overwritten):
    results still match the oracle."""
    tr = tracegen.gen_trace("small_tree")
    ref = oracle.step(tr)
    c = tr["cfg"]
    g = _to_gpu(tr)
    st = A.SpecTrainStep(c.R, c.N, c.d, c.V)
    dH = torch.empty(c.M, c.d, dtype=torch.float32, device="cuda")
    dW = torch.empty(c.V, c.d, dtype=torch.float32, device="cuda")
    st.verify(g["draft"], g["T"], g["parents"], g["num_nodes"])
    st.forward(g["H"], g["W"])
    st.backward(g["H"], g["W"], dH, dW)
    st.backward(g["H"], g["W"], dH, dW)          # second bwd: recompute path
    torch.cuda.synchronize()
    assert _rfro(dW.cpu().numpy(), ref["dW"]) <= GRAD_RFRO and _rfro(dH.cpu().numpy(), ref["dH"]) <= GRAD_RFRO
    st.forward(g["H"], g["W"])
    st.verify(g["draft"], g["T"], g["parents"], g["num_nodes"])   # overwrites the staged partials
    st.backward(g["H"], g["W"], dH, dW)
    torch.cuda.synchronize()
    assert _rfro(dW.cpu().numpy(), ref["dW"]) <= GRAD_RFRO and _rfro(dH.cpu().numpy(), ref["dH"]) <= GRAD_RFRO


def test_staged_dloss_scaling():
    """The upstream gradient g enters the staged rescale and the support fix-up."""
    tr = tracegen.gen_trace("small")
    c = tr["cfg"]
    g = _to_gpu(tr)
    outs = []
    for gv in (None, -2.5):
        st = A.SpecTrainStep(c.R, c.N, c.d, c.V)
        st.verify(g["draft"], g["T"], g["parents"], g["num_nodes"])
        st.forward(g["H"], g["W"])
        dH = torch.empty(c.M, c.d, dtype=torch.float32, device="cuda")
        dW = torch.empty(c.V, c.d, dtype=torch.float32, device="cuda")
        dl = None if gv is None else torch.tensor([gv], device="cuda")
        st.backward(g["H"], g["W"], dH, dW, dloss=dl)
        torch.cuda.synchronize()
        outs.append((dH, dW))
    assert _rfro(outs[1][1].cpu().numpy(), -2.5 * outs[0][1].cpu().numpy()) < 1e-2
    assert _rfro(outs[1][0].cpu().numpy(), -2.5 * outs[0][0].cpu().numpy()) < 1e-2


@pytest.mark.parametrize("group", [3, -2])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(1000, 1300, 192), (256 * 5, 256 * 7, 128)])
def test_gemm_engine_grouped_raster(option, a_mn, b_mn, M, N, K, group):
    """The grouped tile raster of the F4 projections (groups of m-tiles, or of n-tiles when
    negative; ragged last group) covers every tile exactly once: vs PyTorch fp32."""
    option("debug_gemm_group", group)
    test_gemm_engine_vs_torch_fp32(a_mn, b_mn, M, N, K)


@pytest.mark.parametrize("name", ["small", "small_tree", "mid"])
def test_bf16_dw_output(name):
    """§8(b) dW_is_bf16: the dW GEMM's fp32 accumulators rounded once to bf16 (TMA bf16-store
    epilogue); within the north-star bound of the oracle and equal to the fp32 dW rounded."""
    tr = tracegen.gen_trace(name)
    ref = oracle.step(tr)
    c = tr["cfg"]
    g = _to_gpu(tr)
    st = A.SpecTrainStep(c.R, c.N, c.d, c.V)
    st.verify(g["draft"], g["T"], g["parents"], g["num_nodes"])
    st.forward(g["H"], g["W"])
    dH = torch.empty(c.M, c.d, dtype=torch.float32, device="cuda")
    dWb = torch.empty(c.V, c.d, dtype=torch.bfloat16, device="cuda")
    st.backward(g["H"], g["W"], dH, dWb)
    st.forward(g["H"], g["W"])
    dWf = torch.empty(c.V, c.d, dtype=torch.float32, device="cuda")
    st.backward(g["H"], g["W"], dH, dWf)
    torch.cuda.synchronize()
    assert _rfro(dWb.float().cpu().numpy(), ref["dW"]) <= GRAD_RFRO
    assert torch.equal(dWb, dWf.to(torch.bfloat16))
    with pytest.raises(A.AuroraError):   # accumulation into bf16 is not offered
        st.backward(g["H"], g["W"], dH, dWb, accumulate_dW=True)


@pytest.mark.parametrize("kd", [3, 10])
@pytest.mark.parametrize("name", ["tiny", "small", "small_tree", "mid"])
def test_restricted_discard_parity(name, kd):
    """F2, SPEC's restricted-softmax discard loss: DISCARD rows use KL(p~ || q~)
    with q~ the softmax of the support logits (the staged forward's fp32 support logits give
    the support log-sum-exp; the backward keeps dz only on the support), vs oracle O6'."""
    tr = tracegen.gen_trace(name)
    ref = oracle.step_variants(tr, k_discard=kd, discard_loss="restricted")
    out = _run_gpu(tr, k_discard=kd, discard_loss="restricted")
    st = out["st"]
    assert int(st.status.item()) == 0
    np.testing.assert_array_equal(st.row_class.cpu().numpy(), ref["row_class"])
    valid = ref["row_class"] != oracle.PAD
    np.testing.assert_allclose(st.row_loss.cpu().numpy()[valid], ref["row_loss"][valid], rtol=1e-3, atol=2e-4)
    loss = float(st.loss.item())
    assert abs(loss - ref["loss"]) <= LOSS_RTOL * abs(ref["loss"]), (loss, ref["loss"])
    assert _rfro(out["dW"].cpu().numpy(), ref["dW"]) <= GRAD_RFRO
    assert _rfro(out["dH"].cpu().numpy(), ref["dH"]) <= GRAD_RFRO


def test_restricted_discard_needs_the_staged_forward(option):
    option("fwd_stage", 0)
    tr = tracegen.gen_trace("small")
    with pytest.raises(A.AuroraError) as ei:
        _run_gpu(tr, discard_loss="restricted")
    assert ei.value.status == 5

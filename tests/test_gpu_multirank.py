"""Multi-rank parity on ONE GPU through the loopback communicator (-m gpu).

P virtual ranks (one host thread + one CUDA stream each, `aurora_comm_create_loopback`)
run exactly the calls a real rank makes, so the library's multi-rank code executes:
C1 (top-k candidate allgather + global merge), C2 (count allreduce), C3 ((m, s, u, r)
allgather + the P-way row combine), C4 (dH allreduce), C5 (dW allreduce), the F2 triple
merge of the target row statistics and the F3 norm allreduce.

Every rank's results are compared with the single-process f64 oracle on the whole trace
batch: labels and counts bit-exact, loss within 1e-3, dW (vocab shards concatenated) and
dH (request shards concatenated) within 2e-2 relative Frobenius error.
"""
import threading

import numpy as np
import pytest
import torch

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


def _bf16(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def _rfro(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def run_ranks(comms, fn, timeout=600):
    """fn(rank, comm) on its own thread and stream; returns the per-rank results."""
    P = len(comms)
    res, err = [None] * P, [None] * P
    streams = [torch.cuda.Stream() for _ in range(P)]

    def worker(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(streams[r]):
                res[r] = fn(r, comms[r])
                torch.cuda.current_stream().synchronize()
        except BaseException as e:  # noqa: BLE001
            err[r] = e

    ts = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    assert not any(t.is_alive() for t in ts), "virtual ranks deadlocked"
    for e in err:
        if e is not None:
            raise e
    return res


def shard_bounds(n, parts):
    return [(p * n // parts, (p + 1) * n // parts) for p in range(parts)]


def _rank_inputs(tr, vp, dp, rank):
    """This rank's share: requests of its DP slot, vocab slice of its VP slot."""
    c = tr["cfg"]
    q, v = rank // vp, rank % vp
    r0, r1 = shard_bounds(c.R, dp)[q]
    v0, v1 = shard_bounds(c.V, vp)[v]
    rows = slice(r0 * (c.N + 1), r1 * (c.N + 1))
    return dict(r0=r0, r1=r1, v0=v0, v1=v1, rows=rows,
                draft=tr["draft_tokens"][r0:r1],
                parents=None if tr["parents"] is None else tr["parents"][r0:r1],
                num_nodes=None if tr["num_nodes"] is None else tr["num_nodes"][r0:r1],
                T=np.ascontiguousarray(tr["T_bits"][rows, v0:v1]),
                H=np.ascontiguousarray(tr["H_bits"][rows]),
                W=np.ascontiguousarray(tr["W_bits"][v0:v1]))


def run_spec_step(tr, vp, dp, **kw):
    c = tr["cfg"]
    comms = A.aurora_comm_create_loopback(vp * dp, vp, dp)

    def fn(rank, comm):
        x = _rank_inputs(tr, vp, dp, rank)
        R = x["r1"] - x["r0"]
        V_local = x["v1"] - x["v0"]
        st = A.SpecTrainStep(R, c.N, c.d, c.V, V_local=V_local, vocab_offset=x["v0"], comm=comm, **kw)
        T, H, W = _bf16(x["T"]), _bf16(x["H"]), _bf16(x["W"])
        draft = torch.from_numpy(np.ascontiguousarray(x["draft"])).cuda()
        par = None if x["parents"] is None else torch.from_numpy(np.ascontiguousarray(x["parents"])).cuda()
        nn = None if x["num_nodes"] is None else torch.from_numpy(np.ascontiguousarray(x["num_nodes"])).cuda()
        dH = torch.empty(st.M, c.d, dtype=torch.float32, device="cuda")
        dW = torch.empty(V_local, c.d, dtype=torch.float32, device="cuda")
        st.step(draft, T, H, W, dH, dW, par, nn)
        torch.cuda.current_stream().synchronize()
        out = {k: getattr(st, k).cpu().numpy() for k in ("target_argmax", "accepted", "accept_len", "bonus",
                                                         "row_class", "counts", "status", "row_lse", "loss")}
        out.update(dH=dH.cpu().numpy(), dW=dW.cpu().numpy(), x=x)
        return out

    try:
        return run_ranks(comms, fn)
    finally:
        for h in comms:
            A.aurora_comm_destroy(h)


def check_against_oracle(tr, outs, vp, dp, ref):
    c = tr["cfg"]
    for rank, o in enumerate(outs):
        x = o["x"]
        assert int(o["status"][0]) == 0
        np.testing.assert_array_equal(o["target_argmax"], ref["argmax"][x["rows"]])
        np.testing.assert_array_equal(o["accepted"], ref["accepted"][x["r0"]:x["r1"]])
        np.testing.assert_array_equal(o["accept_len"], ref["accept_len"][x["r0"]:x["r1"]])
        np.testing.assert_array_equal(o["bonus"], ref["bonus"][x["r0"]:x["r1"]])
        np.testing.assert_array_equal(o["row_class"], ref["row_class"][x["rows"]])
        assert tuple(o["counts"].tolist()) == tuple(ref["counts"])
        loss = float(o["loss"][0])
        assert abs(loss - ref["loss"]) <= LOSS_RTOL * abs(ref["loss"]), (rank, loss, ref["loss"])
        if "lse" in ref:
            np.testing.assert_allclose(o["row_lse"], ref["lse"][x["rows"]], rtol=2e-5)
    # the members of a VP group hold the same (allreduced) dH; of a DP group the same dW
    for q in range(dp):
        for v in range(1, vp):
            assert np.array_equal(outs[q * vp + v]["dH"], outs[q * vp]["dH"])
    for v in range(vp):
        for q in range(1, dp):
            assert np.array_equal(outs[q * vp + v]["dW"], outs[v]["dW"])
    dH = np.concatenate([outs[q * vp]["dH"] for q in range(dp)])
    dW = np.concatenate([outs[v]["dW"] for v in range(vp)])
    assert dH.shape == (c.M, c.d) and dW.shape == (c.V, c.d)
    assert _rfro(dW, ref["dW"]) <= GRAD_RFRO
    assert _rfro(dH, ref["dH"]) <= GRAD_RFRO


def _ref(tr):
    ref = oracle.step(tr)
    ref["counts"] = ref["targets"]["counts"]
    return ref


@pytest.mark.parametrize("vp", [2, 4, 8])
@pytest.mark.parametrize("name", ["tiny", "small", "small_tree", "mid"])
def test_vocab_parallel(name, vp):
    """VP over P virtual ranks: uneven vocab shards (V // P cuts, not tile multiples),
    candidates of one row spread over shards, ties across shard boundaries (tiny)."""
    tr = tracegen.gen_trace(name)
    check_against_oracle(tr, run_spec_step(tr, vp, 1), vp, 1, _ref(tr))


@pytest.mark.parametrize("dp", [2, 4])
@pytest.mark.parametrize("name", ["small", "small_tree", "mid"])
def test_data_parallel(name, dp):
    """DP over requests: global counts (C2) make the per-term means global, the dW
    allreduce (C5) sums the request shards, the loss allreduce sums the ranks' terms."""
    tr = tracegen.gen_trace(name)
    check_against_oracle(tr, run_spec_step(tr, 1, dp), 1, dp, _ref(tr))


@pytest.mark.parametrize("dp,vp", [(2, 2), (2, 4), (4, 2)])
@pytest.mark.parametrize("name", ["small_tree", "mid"])
def test_dp_x_vp(name, dp, vp):
    """The 2-D layout of the tree config (DP2 x VP4 default)."""
    tr = tracegen.gen_trace(name)
    check_against_oracle(tr, run_spec_step(tr, vp, dp), vp, dp, _ref(tr))


@pytest.mark.parametrize("vp,dp", [(2, 1), (4, 1), (2, 2)])
def test_f2_objectives_multirank(vp, dp):
    """F2 under VP: the per-rank T row triples (max, sum e^{t-m}, sum e^{t-m} t) are
    allgathered and merged in rank order; (m, s, u, r) through C3."""
    tr = tracegen.gen_trace("small")
    kw = dict(accept_loss="rkl", ntp_beta=0.5, k_discard=0)
    ref = oracle.step_variants(tr, **kw)
    check_against_oracle(tr, run_spec_step(tr, vp, dp, **kw), vp, dp, ref)


@pytest.mark.parametrize("opt", [dict(gemm_pair=1, tile_n=224), dict(dz_chunk_bytes=64 << 10), dict(scan_flat=2),
                                 dict(scan_flat=0)])
def test_vocab_parallel_other_launch_configs(opt):
    saved = {k: A.aurora_get_option(k) for k in opt}
    try:
        for k, v in opt.items():
            A.aurora_set_option(k, v)
        tr = tracegen.gen_trace("mid")
        check_against_oracle(tr, run_spec_step(tr, 4, 1), 4, 1, _ref(tr))
    finally:
        for k, v in saved.items():
            A.aurora_set_option(k, v)


def test_loopback_collectives_deterministic():
    """Two runs of the same VP4 step give bit-identical results (ordered sums)."""
    tr = tracegen.gen_trace("small_tree")
    a = run_spec_step(tr, 4, 1)
    b = run_spec_step(tr, 4, 1)
    for x, y in zip(a, b):
        assert np.array_equal(x["dH"], y["dH"]) and np.array_equal(x["dW"], y["dW"])
        assert np.array_equal(x["loss"], y["loss"])


def test_adamw_norm_over_vp_shards():
    """F3 under VP: the global gradient norm is the allreduce of the shards' sums of
    squares; every shard's update equals the oracle's AdamW on the whole tensor."""
    n, vp = 4 * 50021, 4
    inp = tracegen.gen_adamw_inputs(n, steps=2, grad_scale=1e-2)
    cuts = [(a // 4 * 4, b // 4 * 4) for a, b in shard_bounds(n, vp)]
    cuts[-1] = (cuts[-1][0], n)
    comms = A.aurora_comm_create_loopback(vp, vp, 1)
    f32 = lambda x: float(np.float32(x))

    def fn(rank, comm):
        a, b = cuts[rank]
        W = torch.from_numpy(inp["W"][a:b].copy()).cuda()
        opt = A.AdamW(W, lr=1e-3, warmup_steps=0, comm=comm)
        for g in inp["G"]:
            opt.step(torch.from_numpy(g[a:b].copy()).cuda())
        torch.cuda.current_stream().synchronize()
        return W.cpu().numpy(), float(opt.grad_norm.item())

    try:
        outs = run_ranks(comms, fn)
    finally:
        for h in comms:
            A.aurora_comm_destroy(h)
    Wr, mr, vr = inp["W"].astype(np.float64), np.zeros(n), np.zeros(n)
    for step, g in enumerate(inp["G"], start=1):
        Wr, mr, vr, norm = oracle.adamw_step(Wr, mr, vr, g, step, f32(1e-3), beta1=f32(0.9), beta2=f32(0.999),
                                             eps=f32(1e-8), warmup_steps=0)
    for W, gn in outs:
        assert abs(gn - norm) <= 2e-5 * norm
    np.testing.assert_allclose(np.concatenate([W for W, _ in outs]), Wr, rtol=2e-6, atol=1e-9)


@pytest.mark.parametrize("dp,vp", [(2, 1), (4, 1), (2, 2)])
def test_sharded_adamw_dp(dp, vp):
    """F3 DP half: each DP rank's unreduced gradient of its VP slice is reduce-scattered,
    the optimizer state is sharded over the DP group, the norm sums every shard over DP
    and VP, and the updated bf16 lm_head is allgathered.  Against the oracle's AdamW on
    the summed gradient of the whole lm_head, two steps."""
    n_v = 4 * 8 * 1021                      # elements per VP slice (a multiple of 4 * dp)
    n = n_v * vp
    steps = 2
    rng = np.random.default_rng(11)
    W0 = (rng.standard_normal(n) * 0.03).astype(np.float32)
    G = [[(rng.standard_normal(n) * 1e-2).astype(np.float32) for _ in range(dp)] for _ in range(steps)]
    comms = A.aurora_comm_create_loopback(dp * vp, vp, dp)

    def fn(rank, comm):
        q, v = rank // vp, rank % vp
        sl = slice(v * n_v, (v + 1) * n_v)
        Wfull = torch.from_numpy(W0[sl].copy()).cuda()
        Wb = Wfull.to(torch.bfloat16)
        opt = A.ShardedAdamW(Wfull, comm, q, dp, lr=1e-3, warmup_steps=0)
        for t in range(steps):
            opt.step(torch.from_numpy(G[t][q][sl].copy()).cuda(), Wb)
        torch.cuda.current_stream().synchronize()
        return opt.W.cpu().numpy(), Wb.view(torch.int16).cpu().numpy().view(np.uint16), float(opt.grad_norm.item())

    try:
        outs = run_ranks(comms, fn)
    finally:
        for h in comms:
            A.aurora_comm_destroy(h)
    f32 = lambda x: float(np.float32(x))
    Wr, mr, vr = W0.astype(np.float64), np.zeros(n), np.zeros(n)
    for t in range(steps):
        g = G[t][0].copy()                  # the fp32 sum in rank order: the optimizer's input
        for q in range(1, dp):
            g = (g + G[t][q]).astype(np.float32)
        g = g.astype(np.float64)
        Wr, mr, vr, norm = oracle.adamw_step(Wr, mr, vr, g, t + 1, f32(1e-3), beta1=f32(0.9), beta2=f32(0.999),
                                             eps=f32(1e-8), warmup_steps=0)
    sh = n_v // dp
    for rank, (Wsh, Wb, gn) in enumerate(outs):
        q, v = rank // vp, rank % vp
        assert abs(gn - norm) <= 2e-5 * norm
        a = v * n_v + q * sh
        np.testing.assert_allclose(Wsh, Wr[a:a + sh], rtol=2e-6, atol=1e-9)
        # the allgathered bf16 copy is the RNE rounding of the whole updated VP slice
        np.testing.assert_array_equal(Wb, tracegen.f32_to_bf16_bits(Wr[v * n_v:(v + 1) * n_v].astype(np.float32)))

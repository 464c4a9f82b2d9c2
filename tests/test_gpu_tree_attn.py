"""GPU parity of NEXT row F4 (tree attention, aurora_tree_attn_fwd/bwd) against the f64 oracle
(oracle/tree_attention.py) on identical seeded inputs (tracegen.gen_tree_attn).

Tolerances (F4): O is bf16 and P enters the PV product in bf16 (2^-9 relative
rounding), so O is compared at 1e-2 relative Frobenius error per (request, head) slab plus an
elementwise bound; lse is fp32 (ex2.approx, fp32 sums): 2e-3 absolute; the gradients (dQ fp32,
dK/dV bf16, P and dS rounded to bf16 before their products) at the north star's 2e-2 relative
Frobenius error.  Padded rows are exact: O = 0, lse = -inf, dQ = 0, and nobody's key.
"""
import numpy as np
import pytest
import torch

import tracegen
from oracle import tree_attention as TA

pytestmark = pytest.mark.gpu


def _bf(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def _to64(t):
    return t.float().cpu().numpy().astype(np.float64)


def _run(inp, reps=1):
    from paper_2602_06932_b200 import aurora as A
    c = inp["cfg"]
    R, N1 = len(inp["requests"]), c.N + 1
    off = inp["prefix_off"]
    dev = "cuda"
    t = {k: _bf(inp[k + "_bits"]) for k in ["Q", "Kt", "Vt", "Kp", "Vp", "dO"]}
    poff = torch.from_numpy(off.astype(np.int32)).to(dev)
    par = None if inp["parents"] is None else torch.from_numpy(inp["parents"].astype(np.int32)).to(dev)
    nn = None if inp["num_nodes"] is None else torch.from_numpy(inp["num_nodes"].astype(np.int32)).to(dev)
    max_prefix = int(np.max(np.diff(off))) if R else 0
    ta = A.TreeAttention(R, c.N, c.Hq, c.Hkv, c.dh, poff, max_prefix, parents=par, num_nodes=nn)
    outs = []
    for _ in range(reps):
        O = torch.empty_like(t["Q"])
        lse = torch.empty(R, N1, c.Hq, dtype=torch.float32, device=dev)
        dQ = torch.empty(t["Q"].shape, dtype=torch.float32, device=dev)
        g = {k: torch.full_like(t[k], float("nan")) for k in ["Kt", "Vt", "Kp", "Vp"]}
        ta.forward(t["Q"], t["Kt"], t["Vt"], t["Kp"], t["Vp"], O, lse)
        ta.backward(t["Q"], t["Kt"], t["Vt"], t["Kp"], t["Vp"], O, lse, t["dO"], dQ, g["Kt"], g["Vt"], g["Kp"],
                    g["Vp"])
        torch.cuda.synchronize()
        outs.append(dict(O=O, lse=lse, dQ=dQ, dKt=g["Kt"], dVt=g["Vt"], dKp=g["Kp"], dVp=g["Vp"]))
    assert int(ta.status.item()) == 0
    return outs if reps > 1 else outs[0]


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _compare(got, ref, reqs_got, off_got, reqs_ref_off=None):
    """got: device outputs for all requests; ref: oracle on requests reqs_got (in order)."""
    O = _to64(got["O"])[reqs_got]
    lse = got["lse"].cpu().numpy().astype(np.float64)[reqs_got]
    dQ = got["dQ"].cpu().numpy().astype(np.float64)[reqs_got]
    dKt, dVt = _to64(got["dKt"])[reqs_got], _to64(got["dVt"])[reqs_got]
    pidx = np.concatenate([np.arange(off_got[r], off_got[r + 1]) for r in reqs_got])
    dKp, dVp = _to64(got["dKp"])[pidx], _to64(got["dVp"])[pidx]
    fin = np.isfinite(ref["lse"])
    assert np.array_equal(np.isfinite(lse), fin)
    assert np.all(O[~fin] == 0) and np.all(dQ[~fin] == 0)
    np.testing.assert_allclose(lse[fin], ref["lse"][fin], rtol=0, atol=2e-3)
    # O: per (request, head) slab and elementwise
    for r in range(O.shape[0]):
        for h in range(O.shape[2]):
            if np.any(fin[r, :, h]):
                assert _rel(O[r, :, h], ref["O"][r, :, h]) <= 1e-2, (r, h)
    np.testing.assert_allclose(O, ref["O"], rtol=2e-2, atol=2e-2)
    for name, a in [("dQ", dQ), ("dKt", dKt), ("dVt", dVt), ("dKp", dKp), ("dVp", dVp)]:
        if np.linalg.norm(ref[name]) == 0:
            assert np.all(a == 0), name
        else:
            assert _rel(a, ref[name]) <= 2e-2, (name, _rel(a, ref[name]))


# (forward kernel, backward kernel): tree_fwd_tc 2 = one-pass tcgen05, two items per SM (default),
# 3 = one item per SM with deep rings, 1 = two-pass tcgen05, 0 = mma.sync; backward "tc" = tcgen05
# (default), "fused" = mma.sync one-kernel, "split" = the general dQ + dK/dV kernels (used when
# G*(N+1) > 128)
KERNELS = {"tc2_fwd+tc_bwd": (2, "tc"), "tc3_fwd+tc_bwd": (3, "tc"), "tc_fwd+fused_bwd": (1, "fused"),
           "sync_fwd+split_bwd": (0, "split"), "sync_fwd+fused_bwd": (0, "fused"), "sync_fwd+tc_bwd": (0, "tc")}


class _kernels:
    """Context: select the forward / backward kernels through the library options."""

    def __init__(self, fwd_tc, bwd):
        self.fwd_tc, self.bwd = fwd_tc, bwd

    def __enter__(self):
        from paper_2602_06932_b200 import aurora as A
        self.A = A
        self.saved = [A.aurora_get_option(k) for k in ("tree_fwd_tc", "tree_bwd_tc", "tree_bwd_split")]
        A.aurora_set_option("tree_fwd_tc", self.fwd_tc)
        A.aurora_set_option("tree_bwd_tc", 1 if self.bwd == "tc" else 0)
        A.aurora_set_option("tree_bwd_split", 1 if self.bwd == "split" else 0)

    def __exit__(self, *exc):
        for k, v in zip(("tree_fwd_tc", "tree_bwd_tc", "tree_bwd_split"), self.saved):
            self.A.aurora_set_option(k, v)


@pytest.mark.parametrize("kern", list(KERNELS))
@pytest.mark.parametrize("name", ["ta_small", "ta_chain", "ta_gqa8"])
def test_tree_attention_parity(name, kern):
    """Every forward x backward kernel pair against the f64 oracle (O, lse, dQ, dK, dV)."""
    inp = tracegen.gen_tree_attn(name)
    with _kernels(*KERNELS[kern]):
        got = _run(inp)
    ref = TA.fwd_bwd(inp)
    R = len(inp["requests"])
    _compare(got, ref, np.arange(R), inp["prefix_off"])


def test_tree_attention_padded_keys_get_zero_gradients():
    inp = tracegen.gen_tree_attn("ta_small")             # request 2 has num_nodes = 0, request 0 has 6
    got = _run(inp)
    dKt = got["dKt"].float().cpu().numpy()
    assert np.all(dKt[2, 1:] == 0) and np.all(dKt[0, 7:] == 0)
    assert np.all(got["dVt"].float().cpu().numpy()[0, 7:] == 0)


def test_tree_attention_deterministic():
    inp = tracegen.gen_tree_attn("ta_gqa8")
    a, b = _run(inp, reps=2)
    for k in a:
        assert torch.equal(a[k], b[k]), k


@pytest.mark.parametrize("kern", ["tc2_fwd+tc_bwd", "tc3_fwd+tc_bwd", "sync_fwd+fused_bwd"])
@pytest.mark.parametrize("name,sample", [("ta_llama", [0, 37, 63]), ("ta_tree", [0, 511, 1023])])
def test_tree_attention_full_size_sampled(name, sample, kern):
    """Full BASELINE sizes in the bench's launch configuration; the oracle recomputes a sample of
    requests (each request is independent, so the sample is exact)."""
    inp = tracegen.gen_tree_attn(name)
    with _kernels(*KERNELS[kern]):
        got = _run(inp)
    ref = TA.fwd_bwd(tracegen.gen_tree_attn(name, requests=sample))
    _compare(got, ref, np.asarray(sample), inp["prefix_off"])
    # every prefix gradient row of the whole batch was written (no NaN sentinel left)
    assert not torch.isnan(got["dKp"]).any() and not torch.isnan(got["dVp"]).any()


def test_tree_attention_errors():
    from paper_2602_06932_b200 import aurora as A
    inp = tracegen.gen_tree_attn("ta_chain")
    c = inp["cfg"]
    R, N1 = c.R, c.N + 1
    poff = torch.from_numpy(inp["prefix_off"].astype(np.int32)).cuda()
    t = {k: _bf(inp[k + "_bits"]) for k in ["Q", "Kt", "Vt", "Kp", "Vp"]}
    O = torch.empty_like(t["Q"])
    lse = torch.empty(R, N1, c.Hq, dtype=torch.float32, device="cuda")
    with pytest.raises(A.AuroraError):               # dh != 128: UNSUPPORTED, nothing enqueued
        A.TreeAttention(R, c.N, c.Hq, c.Hkv, 64, poff, 300).forward(t["Q"], t["Kt"], t["Vt"], t["Kp"], t["Vp"],
                                                                    O, lse)
    # malformed parents (a parent after its child): STRUCTURE bit, the affected rows padded
    bad = torch.tensor([[-1, 0, 5, 1, 2]] * R, dtype=torch.int32, device="cuda")
    ta = A.TreeAttention(R, c.N, c.Hq, c.Hkv, c.dh, poff, 300, parents=bad)
    ta.forward(t["Q"], t["Kt"], t["Vt"], t["Kp"], t["Vp"], O, lse)
    torch.cuda.synchronize()
    assert int(ta.status.item()) & A.STATUS_STRUCTURE
    assert torch.isneginf(lse[:, 3]).all() and torch.isfinite(lse[:, :3]).all()
    # a prefix longer than max_prefix: RANGE bit
    ta = A.TreeAttention(R, c.N, c.Hq, c.Hkv, c.dh, poff, 10)
    ta.forward(t["Q"], t["Kt"], t["Vt"], t["Kp"], t["Vp"], O, lse)
    torch.cuda.synchronize()
    assert int(ta.status.item()) & A.STATUS_RANGE


@pytest.mark.parametrize("name,theta", [("ta_small", 500000.0), ("ta_gqa8", 1000000.0), ("ta_chain", 10000.0)])
def test_tree_rope_parity(name, theta):
    """F4-R6: tree positions + rotate-half RoPE against the oracle (bf16 in place: one bf16
    rounding of the rotated value; f32 inverse on the rotated values: round trip)."""
    from paper_2602_06932_b200 import aurora as A
    inp = tracegen.gen_tree_attn(name)
    c = inp["cfg"]
    R = len(inp["requests"])
    off = inp["prefix_off"]
    poff = torch.from_numpy(off.astype(np.int32)).cuda()
    par = None if inp["parents"] is None else torch.from_numpy(inp["parents"].astype(np.int32)).cuda()
    nn = None if inp["num_nodes"] is None else torch.from_numpy(inp["num_nodes"].astype(np.int32)).cuda()
    ta = A.TreeAttention(R, c.N, c.Hq, c.Hkv, c.dh, poff, int(np.diff(off).max()), parents=par, num_nodes=nn)
    Q, Kt = _bf(inp["Q_bits"]), _bf(inp["Kt_bits"])
    pos = TA.tree_rope_positions(off, inp["parents"], inp["num_nodes"], R, c.N)
    q64, k64 = TA.bf16_bits_to_f64(inp["Q_bits"]), TA.bf16_bits_to_f64(inp["Kt_bits"])
    ref_q, ref_k = TA.rope(q64, pos, theta), TA.rope(k64, pos, theta)
    Qf, Ktf = Q.float().clone(), Kt.float().clone()
    ta.rope(Q, Kt, theta=theta)
    ta.rope(Qf, Ktf, theta=theta)
    torch.cuda.synchronize()
    assert int(ta.status.item()) == 0
    for got, ref in [(Q, ref_q), (Kt, ref_k)]:
        g = _to64(got)
        np.testing.assert_allclose(g, ref, rtol=2 ** -8, atol=1e-5)           # one bf16 rounding
    np.testing.assert_allclose(Qf.cpu().numpy(), ref_q, rtol=1e-5, atol=1e-5)   # f32 storage
    np.testing.assert_allclose(Ktf.cpu().numpy(), ref_k, rtol=1e-5, atol=1e-5)
    # padded rows untouched, inverse restores the input (f32)
    pad = pos < 0
    if pad.any():
        assert np.array_equal(_to64(Q)[pad], q64[pad])
    ta.rope(Qf, Ktf, theta=theta, inverse=True)
    torch.cuda.synchronize()
    np.testing.assert_allclose(Qf.cpu().numpy(), q64, rtol=1e-5, atol=2e-5)
    np.testing.assert_allclose(Ktf.cpu().numpy(), k64, rtol=1e-5, atol=2e-5)


def test_malformed_prefix_offsets_flag_range_without_oob():
    """prefix_off entries outside [0, prefix_total] (or decreasing) set the RANGE
    bit and make that request's prefix empty — Kp/Vp are never read or written out of bounds
    (the guard bands around them stay untouched) and every output stays finite."""
    from paper_2602_06932_b200 import aurora as A
    inp = tracegen.gen_tree_attn("ta_small")
    c = inp["cfg"]
    R, N1 = len(inp["requests"]), c.N + 1
    off = inp["prefix_off"].astype(np.int32).copy()
    total = int(off[-1])
    bad = off.copy()
    bad[2] = total + 500                      # request 1 ends beyond Kp, request 2 starts there
    dev = "cuda"
    t = {k: _bf(inp[k + "_bits"]) for k in ["Q", "Kt", "Vt", "dO"]}
    guard = 4096
    Kp_all = torch.zeros(total + 2 * guard, c.Hkv, c.dh, dtype=torch.bfloat16, device=dev)
    Vp_all = torch.zeros_like(Kp_all)
    Kp_all[guard:guard + total] = _bf(inp["Kp_bits"])
    Vp_all[guard:guard + total] = _bf(inp["Vp_bits"])
    Kp, Vp = Kp_all[guard:guard + total], Vp_all[guard:guard + total]
    dKp_all = torch.full_like(Kp_all, 7.0)
    dVp_all = torch.full_like(Kp_all, 7.0)
    par = None if inp["parents"] is None else torch.from_numpy(inp["parents"].astype(np.int32)).to(dev)
    nn = None if inp["num_nodes"] is None else torch.from_numpy(inp["num_nodes"].astype(np.int32)).to(dev)
    ta = A.TreeAttention(R, c.N, c.Hq, c.Hkv, c.dh, torch.from_numpy(bad).to(dev), int(np.max(np.diff(off))),
                         parents=par, num_nodes=nn, prefix_total=total)
    O = torch.empty_like(t["Q"])
    lse = torch.empty(R, N1, c.Hq, dtype=torch.float32, device=dev)
    dQ = torch.empty(t["Q"].shape, dtype=torch.float32, device=dev)
    dKt, dVt = torch.empty_like(t["Kt"]), torch.empty_like(t["Vt"])
    ta.forward(t["Q"], t["Kt"], t["Vt"], Kp, Vp, O, lse)
    ta.backward(t["Q"], t["Kt"], t["Vt"], Kp, Vp, O, lse, t["dO"], dQ, dKt, dVt, dKp_all[guard:guard + total],
                dVp_all[guard:guard + total])
    torch.cuda.synchronize()
    assert int(ta.status.item()) & A.STATUS_RANGE
    assert torch.isfinite(O.float()).all() and torch.isfinite(dQ).all()
    for g in (dKp_all, dVp_all):
        assert bool((g[:guard].float() == 7.0).all()) and bool((g[guard + total:].float() == 7.0).all())


@pytest.mark.parametrize("kern", ["tc2_fwd+tc_bwd", "tc3_fwd+tc_bwd", "sync_fwd+fused_bwd"])
@pytest.mark.parametrize("p_len", [0, 64, 128])
def test_tree_attention_prefix_edge_lengths(kern, p_len):
    """Every request's prefix empty (no Kp / Vp at all: the tensor maps fall back to the tree
    keys) or exactly one / two full 64-key tiles (no partial prefix tile), against the oracle."""
    cfg = tracegen.TreeAttnConfig(f"ta_edge{p_len}", R=5, N=9, Hq=16, Hkv=4, dh=128, p_min=p_len, p_max=p_len,
                                  seed=3100 + p_len, tree=True, beam=3)
    inp = tracegen.gen_tree_attn(cfg)
    assert int(inp["prefix_off"][-1]) == 5 * p_len
    with _kernels(*KERNELS[kern]):
        got = _run(inp)
    ref = TA.fwd_bwd(inp)
    _compare(got, ref, np.arange(5), inp["prefix_off"])

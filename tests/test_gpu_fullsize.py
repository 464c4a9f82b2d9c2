"""Full-size GPU parity at the bench's headline workload and adversarial scan rows at full
vocabulary (-m gpu).

* qwen3 (BASELINE.json configs[2], the workload `bench.py` times by default, in the same
  launch configuration): labels bit-exact on every row, sup_idx / sup_p / w / H~ on every
  row, the total loss within 1e-3 against the oracle's f64 lse of all 1792 rows, dH on
  sampled rows and dW on vocabulary slices (head, middle, the ragged tail and the slices
  holding sampled support tokens) within 2e-2 relative Frobenius error — O5 evaluated by
  `oracle.loss_bwd_sampled`, the same definitions as the full backward.
* A2 edge cases at V = 151,936: constant rows, exact maxima straddling every possible
  segment boundary of the multi-CTA scan, +-0 at the maximum, all-negative rows, and ties
  at the 10th place spread across segments — compared bit-exact with `oracle.target_scan`
  (value desc, index asc; numeric compare, -0 == +0, reading Q8).
"""
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


@pytest.fixture(scope="module")
def qwen3_run():
    tr = tracegen.gen_trace("qwen3")
    c = tr["cfg"]
    st = A.SpecTrainStep(c.R, c.N, c.d, c.V)
    T, H, W = _bf16(tr["T_bits"]), _bf16(tr["H_bits"]), _bf16(tr["W_bits"])
    draft = torch.from_numpy(tr["draft_tokens"]).cuda()
    dH = torch.empty(c.M, c.d, dtype=torch.float32, device="cuda")
    dW = torch.empty(c.V, c.d, dtype=torch.float32, device="cuda")
    st.step(draft, T, H, W, dH, dW)
    torch.cuda.synchronize()
    del T
    out = dict(tr=tr, st=st, dH=dH.cpu().numpy(), dW=dW, W=W)
    # oracle: scan + verify + targets on every row, lse of every row (f64)
    Tb = tr["T_bits"]
    M = c.M
    am = np.empty(M, dtype=np.int64)
    topk = np.empty((M, 10), dtype=np.int64)
    for m0 in range(0, M, 256):
        a, t, nf = oracle.target_scan(oracle.bf16_bits_to_f64(Tb[m0:m0 + 256]), 10)
        assert not nf
        am[m0:m0 + 256], topk[m0:m0 + 256] = a, t
    lab = oracle.verify(tr["draft_tokens"], None, None, am)
    tg = oracle.row_targets(lab["row_class"], lambda m: oracle.bf16_bits_to_f64(Tb[m]), topk)
    H64 = oracle.bf16_bits_to_f64(tr["H_bits"])
    fw = oracle.loss_fwd(H64, tr["W_bits"], tg)
    out.update(am=am, lab=lab, tg=tg, fw=fw, H64=H64)
    return out


def test_qwen3_labels_and_targets_every_row(qwen3_run):
    r = qwen3_run
    st, lab, tg = r["st"], r["lab"], r["tg"]
    assert int(st.status.item()) == 0
    np.testing.assert_array_equal(st.target_argmax.cpu().numpy(), r["am"])
    np.testing.assert_array_equal(st.accepted.cpu().numpy(), lab["accepted"])
    np.testing.assert_array_equal(st.accept_len.cpu().numpy(), lab["accept_len"])
    np.testing.assert_array_equal(st.bonus.cpu().numpy(), lab["bonus"])
    np.testing.assert_array_equal(st.row_class.cpu().numpy(), lab["row_class"])
    assert tuple(st.counts.cpu().tolist()) == tuple(tg["counts"])
    sup, sp = st.sup_idx.cpu().numpy(), st.sup_p.cpu().numpy()
    w, Hh = st.row_w.cpu().numpy(), st.row_H.cpu().numpy()
    for m in range(r["tr"]["M"]):
        k = len(tg["sup_idx"][m])
        np.testing.assert_array_equal(sup[m, :k], tg["sup_idx"][m])
        np.testing.assert_allclose(sp[m, :k], tg["sup_p"][m], rtol=2e-6, atol=1e-7)
        assert abs(w[m] - tg["w"][m]) <= 1e-6 * abs(tg["w"][m]) + 1e-12
        assert abs(Hh[m] - tg["H"][m]) <= 1e-5


def test_qwen3_loss_and_lse_every_row(qwen3_run):
    r = qwen3_run
    st, fw = r["st"], r["fw"]
    np.testing.assert_allclose(st.row_lse.cpu().numpy(), fw["lse"], rtol=2e-5)
    valid = r["lab"]["row_class"] != oracle.PAD
    np.testing.assert_allclose(st.row_loss.cpu().numpy()[valid], fw["row_loss"][valid], rtol=1e-3, atol=1e-3)
    loss = float(st.loss.item())
    assert abs(loss - fw["loss"]) <= LOSS_RTOL * abs(fw["loss"]), (loss, fw["loss"])


def test_qwen3_grads_sampled(qwen3_run):
    """dH on 48 rows (both domains of the ordered stream, ACCEPT and DISCARD rows) and dW on
    vocabulary slices, each against the oracle's O5 at full V / full M."""
    r = qwen3_run
    tr, tg = r["tr"], r["tg"]
    M, V = tr["M"], tr["V"]
    rng = np.random.default_rng(7)
    rows = np.sort(rng.choice(M, size=48, replace=False))
    # slices: head, a middle slice, the ragged tail, and 512-column slices around three
    # support tokens (the columns where the -p~ term lands)
    sup_cols = [int(tg["sup_idx"][int(m)][0]) for m in rows[:3] if len(tg["sup_idx"][int(m)])]
    ranges = {(0, 512), (V // 2 - 256, V // 2 + 256), (V - 700, V)}
    for j in sup_cols:
        v0 = max(0, min(V - 512, j - 256))
        ranges.add((v0, v0 + 512))
    ranges = sorted(ranges)
    ref = oracle.loss_bwd_sampled(r["H64"], tr["W_bits"], tg, r["fw"]["lse"], rows, ranges)
    assert _rfro(r["dH"][rows], ref["dH"]) <= GRAD_RFRO
    dW = r["dW"]
    for v0, v1 in ranges:
        got = dW[v0:v1].cpu().numpy()
        assert _rfro(got, ref["dW"][(v0, v1)]) <= GRAD_RFRO, (v0, v1)


# ----------------------------------------------------------------------------- A2 edge cases
def _bits(x):
    return tracegen.f32_to_bf16_bits(np.asarray(x, dtype=np.float32))


def _adversarial_rows(V, seed):
    """Rows whose argmax / top-10 sit where a segmented scan can get them wrong."""
    rng = np.random.default_rng(seed)
    rows = []
    base = lambda: rng.normal(-5.0, 1.0, size=V).astype(np.float32)   # all negative
    # every segment boundary a scan with 1..32 segments of 8-aligned length could use
    bounds = sorted({((V + n - 1) // n + 7) // 8 * 8 * k for n in range(1, 33) for k in range(1, n)} - {0})
    bounds = [b for b in bounds if 0 < b < V]
    rows.append(np.ones(V, np.float32))                          # constant row: ids 0..9
    z = np.zeros(V, np.float32)
    z[rng.random(V) < 0.5] = -0.0                                # constant +-0
    rows.append(z)
    for b in bounds[::max(1, len(bounds) // 24)]:                # exact max straddling a boundary
        t = base()
        t[b - 1] = t[b] = 3.0
        rows.append(t)
        t = base()                                               # 12-way tie around it (10th place)
        t[max(0, b - 6):b + 6] = 2.5
        rows.append(t)
    t = base()
    t[0] = t[V - 1] = 1.0                                        # first and last column
    rows.append(t)
    t = base()
    t[V - 1] = 4.0                                               # max in the ragged tail
    rows.append(t)
    t = base()
    t[777], t[70001] = -0.0, 0.0                                 # +-0 at the maximum
    rows.append(t)
    t = base()
    t[123456], t[5] = 0.0, -0.0
    rows.append(t)
    t = base()                                                   # 10th-place tie across segments
    t[rng.choice(V, 9, replace=False)] = 6.0
    t[np.array([b for b in bounds[:40:3]])] = 1.25
    rows.append(t)
    t = np.full(V, -3.0e38, np.float32)                          # huge negatives, one tie pair
    t[[4000, 150000]] = -1.0e38
    rows.append(t)
    return np.stack(rows)


SCAN_MODES = {"flat": (2, 0), "seg": (0, 0), "ring": (0, 1)}   # (scan_flat, scan_ring)


def _with_scan_mode(mode, fn, *a):
    saved = [A.aurora_get_option("scan_flat"), A.aurora_get_option("scan_ring")]
    A.aurora_set_option("scan_flat", SCAN_MODES[mode][0])
    A.aurora_set_option("scan_ring", SCAN_MODES[mode][1])
    try:
        fn(*a)
    finally:
        A.aurora_set_option("scan_flat", saved[0])
        A.aurora_set_option("scan_ring", saved[1])


@pytest.mark.parametrize("mode", list(SCAN_MODES))
@pytest.mark.parametrize("R,N", [(1, 1), (8, 7), (64, 6)])
def test_scan_adversarial_rows_full_vocab(R, N, mode):
    """Bit-exact argmax and top-10 set (k_accept = k_discard = 10 exposes the whole list)
    at V = 151,936 for three row counts (several segment counts per row), for the default
    load-balanced scan (scan_flat), the (row, segment) scan and the TMA-ring scan."""
    _with_scan_mode(mode, _scan_adversarial, R, N)


def _flat_piece_bounds(M, V):
    """Columns where the flat scan's warp ranges start inside each row (the split the library
    documents for option scan_flat: W = min(2 * 148 * 8, NV / 64) equal ranges of the NV =
    M * V / 8 row-major vectors, range g starting at vector g * NV // W)."""
    V8 = V // 8
    NV = M * V8
    W = max(1, min(2 * 148 * 8, NV // 64))
    out = [[] for _ in range(M)]
    for g in range(1, W):
        s = g * NV // W
        r, c = divmod(s, V8)
        if c:
            out[r].append(8 * c)
    return out


@pytest.mark.parametrize("R,N", [(8, 7), (64, 6), (128, 6)])
def test_scan_flat_range_boundaries(R, N):
    """The load-balanced scan cuts rows at warp-range boundaries: exact maxima and 10th-place
    ties straddling those cuts, maxima as the first / last column of a piece, bit-exact against
    the oracle."""
    V = 151936
    M = R * (N + 1)
    rng = np.random.default_rng(M + 1)
    T32 = rng.normal(-5.0, 1.0, size=(M, V)).astype(np.float32)
    cuts = _flat_piece_bounds(M, V)
    for m in range(M):
        for j, b in enumerate(cuts[m]):
            kind = (m + j) % 4
            if kind == 0:
                T32[m, b - 1] = T32[m, b] = 3.0                  # tied maximum across the cut
            elif kind == 1:
                T32[m, rng.choice(V, 9, replace=False)] = 6.0    # 10th place tied across the cut
                T32[m, max(0, b - 6):b + 6] = 2.5
            elif kind == 2:
                T32[m, b] = 4.0                                  # max = first column of a piece
            else:
                T32[m, b - 1] = 4.0                              # max = last column of a piece
    _with_scan_mode("flat", _scan_check, R, N, T32)


def _scan_adversarial(R, N):
    V = 151936
    M = R * (N + 1)
    rows = _adversarial_rows(V, seed=M)
    reps = (M + len(rows) - 1) // len(rows)
    _scan_check(R, N, np.concatenate([rows] * reps)[:M])


def _scan_check(R, N, T32, k=10):
    M, V = T32.shape
    Tb = _bits(T32)
    T64 = oracle.bf16_bits_to_f64(Tb)
    am, topk, nf = oracle.target_scan(T64, k)
    assert not nf
    draft = torch.zeros(R, N, dtype=torch.int32, device="cuda")
    st = A.SpecTrainStep(R, N, 64, V, k_accept=k, k_discard=k)
    st.verify(draft, _bf16(Tb))
    torch.cuda.synchronize()
    assert int(st.status.item()) == 0
    np.testing.assert_array_equal(st.target_argmax.cpu().numpy(), am)
    sup = st.sup_idx.cpu().numpy()
    for m in range(M):
        np.testing.assert_array_equal(sup[m, :k], np.sort(topk[m]), err_msg=f"row {m}")


@pytest.mark.parametrize("mode", ["flat", "seg"])
def test_scan_top16_full_vocab(mode):
    """The largest dense list (k_accept = k_discard = 16 = AURORA_MAX_K): every row's top-16 set
    and argmax bit-exact at V = 151,936, bf16-quantised N(0, 4) rows with a 40-way tie across the
    16th place in some rows."""
    R, N, V = 16, 6, 151936
    rng = np.random.default_rng(32)
    T32 = (rng.standard_normal((R * (N + 1), V)) * 2.0).astype(np.float32)
    for m in range(0, R * (N + 1), 3):
        T32[m, rng.choice(V, 40, replace=False)] = 9.0
    _with_scan_mode(mode, _scan_check, R, N, T32, 16)

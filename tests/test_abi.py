"""C-ABI library loads and exports every symbol include/aurora.h declares; host-side
validation returns the documented status without touching a GPU (-m "not gpu")."""
import ctypes as C
import os
import re

import pytest

from paper_2602_06932_b200 import aurora as A
from paper_2602_06932_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    build()
    return A.lib()


def _declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "aurora.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(aurora_[a-z_]+)\s*\(", hdr)))


def test_exports_every_declared_symbol(L):
    declared = _declared_symbols()
    assert len(declared) >= 12
    assert sorted(A.EXPORTS) == declared
    for name in declared:
        assert hasattr(L, name), name


def test_status_strings_and_build_info(L):
    for s in range(9):
        assert L.aurora_status_string(s)
    assert b"sm_100a" in L.aurora_build_info()


def test_workspace_size_monotone(L):
    cfg = A.aurora_loss_cfg_t(1, 10, 1.0, 0, 0)
    small = A.aurora_workspace_size(A.OP_ALL, 20, 64, 1000, cfg)
    big = A.aurora_workspace_size(A.OP_ALL, 384, 4096, 128256, cfg)
    assert 0 < small < big
    assert A.aurora_workspace_size(A.OP_ALL, 0, 64, 1000, cfg) == 0
    # bwd dLogits chunk never exceeds the dz_chunk_bytes budget (+ split-K partials, alignment)
    saved = A.aurora_get_option("dz_chunk_bytes")
    try:
        for budget in (1 << 31, 16 << 20):
            A.aurora_set_option("dz_chunk_bytes", budget)
            bwd = A.aurora_workspace_size(A.OP_BWD, 384, 4096, 128256, cfg)
            assert bwd < min(budget, 384 * 128256 * 2) + 256 * 384 * 2 + 8 * 384 * 4096 * 4 + (1 << 20)
    finally:
        A.aurora_set_option("dz_chunk_bytes", saved)


def test_host_validation_without_gpu(L):
    cfg = A.aurora_loss_cfg_t(1, 10, 1.0, 0, 0)
    lab = A.aurora_labels_t()
    # NULL trace -> invalid arg, nothing enqueued (no CUDA call happens)
    assert L.aurora_verify_labels(None, C.byref(cfg), C.byref(lab), None, 0, None, None) == 1
    # F2 objectives need the dense target row: unsupported with the sparse payload
    lab_ok = A.aurora_labels_t(10, 16, 16, 16, 16, 16, 16, 16, 16, 16, 16, 16)
    tk = A.aurora_trace_topk_t(4, 4, 16, None, None, 16, 16, 64, 1000)
    for cfg_f2 in (A.aurora_loss_cfg_t(1, 0, 1.0, 0, 0), A.aurora_loss_cfg_t(1, 10, 1.0, 0, 0, 1, 0.5)):
        assert L.aurora_verify_labels_topk(C.byref(tk), C.byref(cfg_f2), C.byref(lab_ok), None, 0, None, None) == 5
    # invalid objective settings: NTP without RKL, unknown accept_loss, negative beta
    t = A.aurora_trace_t(4, 4, 16, 0, 0, 16, 1000, 1000, 1000, 0)
    for bad in (A.aurora_loss_cfg_t(1, 10, 1.0, 0, 0, 0, 0.5), A.aurora_loss_cfg_t(1, 10, 1.0, 0, 0, 2, 0.0),
                A.aurora_loss_cfg_t(1, 10, 1.0, 0, 0, 1, -1.0)):
        assert L.aurora_verify_labels(C.byref(t), C.byref(bad), C.byref(lab_ok), None, 0, None, None) == 1
    # N > 32
    t2 = A.aurora_trace_t(4, 33, 16, 0, 0, 16, 1000, 1000, 1000, 0)
    assert L.aurora_verify_labels(C.byref(t2), C.byref(cfg), C.byref(lab), None, 0, None, None) == 1
    # fwd with d not a multiple of 64
    assert L.aurora_spec_loss_fwd(16, 16, 20, 100, 1000, 0, C.byref(lab), 16, None, 16, None, 0, None, None) == 1
    # bf16 dW output: supported, but not with accumulation (host-detectable, nothing enqueued)
    lab2 = A.aurora_labels_t(10, 16, 16, 16, 16, 16, 16, 16, 16, 16, 16, 16)
    assert L.aurora_spec_loss_bwd(16, 16, 20, 64, 1000, 0, C.byref(lab2), 16, None, 16, 16, 1, 1, 16, 1 << 30,
                                  None, None) == 5
    # missing workspace
    assert L.aurora_spec_loss_fwd(16, 16, 20, 64, 1000, 0, C.byref(lab2), 16, None, 16, None, 0, None, None) == 6
    # comm argument validation
    h = C.c_void_p()
    assert L.aurora_comm_create(None, 2, 0, 1, 2, C.byref(h)) == 1
    assert L.aurora_comm_create(C.create_string_buffer(128), 2, 0, 3, 1, C.byref(h)) == 1


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle."""
    pkg = os.path.join(ROOT, "paper_2602_06932_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith(".py"):
                src = open(os.path.join(dp, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_options_validate_host_side(L):
    """Execution options are host state: valid values round-trip, invalid ones are rejected."""
    for name, good, bad in [("gemm_pair", (0, 1, 2), (3, -1)), ("bwd_mode", (0, 1), (2,)),
                            ("bwd_concurrent", (0, 1), (2,)), ("tile_n", (0, 256, 224, 192), (128, 200, 512)),
                            ("dz_chunk_bytes", (1 << 20, 1 << 31), (0, -5)), ("scan_ctas", (1, 2, 16), (0, 17)),
                            ("dw_resident", (0, 1), (2,)), ("scan_flat", (0, 1, 2), (3,)),
                            ("tree_fwd_tc", (0, 1, 3, 2), (4, 5, -1)), ("tree_bwd_tc", (0, 1), (2,)),
                            ("tree_bwd_split", (1, 0), (2,))]:
        saved = A.aurora_get_option(name)
        try:
            for v in good:
                A.aurora_set_option(name, v)
                assert A.aurora_get_option(name) == v
            for v in bad:
                with pytest.raises(Exception):
                    A.aurora_set_option(name, v)
                assert A.aurora_get_option(name) == good[-1]
        finally:
            A.aurora_set_option(name, saved)
    assert A.aurora_get_option("no_such_option") == -1


def test_documented_option_defaults(L):
    """The defaults aurora.h documents (read in a fresh process: options are process-wide and the
    environment can override them): tcgen05 tree attention, load-balanced scan where it pays,
    serial per-chunk backward, auto CTA pairs / tile width, 16 GiB dZ^T chunk budget."""
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if not k.startswith("AURORA_")}
    code = ("from paper_2602_06932_b200 import aurora as A; A.lib(); print([A.aurora_get_option(n) for n in "
            "('tree_fwd_tc', 'tree_bwd_tc', 'tree_bwd_split', 'scan_flat', 'bwd_mode', 'bwd_concurrent', "
            "'gemm_pair', 'tile_n', 'dz_chunk_bytes', 'dw_resident')])")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().splitlines()[-1] == str([2, 1, 0, 1, 0, 0, 0, 0, 16 << 30, 0])


def test_tree_attn_host_validation_without_gpu(L):
    """F4 entry points reject bad configurations before any CUDA call (nothing enqueued)."""
    ok = dict(R=4, N=5, Hq=32, Hkv=8, dh=128, max_prefix=100, prefix_total=300, prefix_off=16)
    ta = lambda **kw: A.aurora_tree_attn_t(**{**ok, **kw})
    P = [16] * 5                                     # Q, Kt, Vt, Kp, Vp (aligned dummies)
    f = lambda t, ptrs=P, o=16, lse=16: L.aurora_tree_attn_fwd(C.byref(t), *ptrs, o, lse, None)
    assert L.aurora_tree_attn_fwd(None, *P, 16, 16, None) == 1
    assert f(ta(dh=64)) == 5                         # head dim 128 only
    assert f(ta(N=33)) == 5                          # N <= 32
    assert f(ta(Hq=30)) == 1                         # Hq % Hkv
    assert f(ta(Hq=64, Hkv=1, N=5)) == 5             # G * (N + 1) = 384 > 256 rows per KV head
    assert f(ta(R=0)) == 1
    assert f(ta(prefix_off=None)) == 1
    assert f(ta(), ptrs=[16, 16, 16, None, 16]) == 1  # prefix K missing while max_prefix > 0
    assert f(ta(), ptrs=[24, 16, 16, 16, 16]) == 1    # Q not 16-B aligned
    assert f(ta(), o=None) == 1
    t = ta()
    need = L.aurora_tree_attn_workspace_size(C.byref(t))
    assert need >= 4 * 6 * 32 * 4
    b = lambda t, ws_bytes, dq=16: L.aurora_tree_attn_bwd(C.byref(t), *P, 16, 16, 16, dq, 16, 16, 16, 16, 16,
                                                          ws_bytes, None)
    assert b(t, need - 1) == 6                       # workspace too small
    assert b(t, need, dq=None) == 1
    assert b(ta(dh=64), need) == 5


def test_draft_layer_host_validation_without_gpu(L):
    """F4 draft layer: bad configurations and missing buffers return before any CUDA call."""
    ta = A.aurora_tree_attn_t(R=4, N=5, Hq=32, Hkv=8, dh=128, max_prefix=100, prefix_total=300, prefix_off=16)
    cfg = A.aurora_draft_layer_t(ta, 4096, 14336, 500000.0, 1e-6)
    W = A.aurora_draft_weights_t(*([16] * 12))
    need = L.aurora_draft_layer_workspace_size(C.byref(cfg))
    assert need > 24 * 4096 * 4
    f = lambda c, w=W, ws=need, h=16: L.aurora_draft_layer_fwd(C.byref(c), C.byref(w), h, 16, 16, 16, 16, 16, ws, None)
    assert f(A.aurora_draft_layer_t(ta, 4100, 14336, 5e5, 1e-6)) == 1                                   # d % 8
    assert f(A.aurora_draft_layer_t(ta, 4096, 14336, 5e5, 0.0)) == 1                                    # eps
    assert f(A.aurora_draft_layer_t(A.aurora_tree_attn_t(R=4, N=5, Hq=32, Hkv=8, dh=64, prefix_off=16), 4096,
                                    14336, 5e5, 1e-6)) == 5                                             # dh
    assert f(cfg, w=A.aurora_draft_weights_t(*([16] * 11 + [None]))) == 1                              # w_final
    assert f(cfg, h=None) == 1
    assert f(cfg, ws=need - 1) == 6
    G = A.aurora_draft_grads_t(*([16] * 12))
    b = lambda g: L.aurora_draft_layer_bwd(C.byref(cfg), C.byref(W), 16, 16, 16, 16, 16, C.byref(g), 16, 16, 16, 16,
                                           16, need, None)
    assert b(A.aurora_draft_grads_t(*([16] * 11 + [None]))) == 1


def test_speculator_params_layout():
    """SpeculatorParams views tile the flat buffers exactly (no overlap, no gap); the norm weights
    are fp32 views of the master (the kernels read them), the matrices bf16 views of the copy."""
    import numpy as np
    import torch
    sp = A.SpeculatorParams(d=64, I=96, Hq=2, Hkv=1, dh=128, V=300, device="cpu")
    names = [n for n, _ in sp.shapes]
    total = sum(int(np.prod(s)) for _, s in sp.shapes)
    assert sp.master.numel() == sp.bf.numel() == sp.grad.numel() == total
    starts = sorted((sp.M[n].data_ptr() - sp.master.data_ptr()) // 4 for n in names)
    sizes = {(sp.M[n].data_ptr() - sp.master.data_ptr()) // 4: sp.M[n].numel() for n in names}
    pos = 0
    for st in starts:
        assert st == pos
        pos += sizes[st]
    assert pos == total
    for n in ("we", "wh", "wpost", "wfinal"):
        assert sp.W[n].dtype == torch.float32 and sp.W[n].data_ptr() == sp.M[n].data_ptr()
    for n in ("Wfc", "Wq", "Wd"):
        assert sp.W[n].dtype == torch.bfloat16 and sp.W[n].is_contiguous()
    assert sp.W_lm.shape == (300, 64) and sp.dW_lm.shape == (300, 64) and "W_lm" not in sp.W
    sp.load({"wh": np.full(64, 2.0), "Wq": np.ones((256, 128))})
    assert float(sp.W["wh"].sum()) == 128.0 and float(sp.W["Wq"].float().sum()) == 256 * 128

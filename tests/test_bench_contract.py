"""CPU checks of bench.py's measurement bookkeeping: the roofline picks
the dominant phase, uses the bound (tensor or HBM) that the algorithmic work implies, and
reports traffic only for the workload the committed ncu capture ran."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_roofline_dominant_phase_and_bounds(bench):
    import tracegen
    cfg = tracegen.CONFIGS["llama"]
    steps = 10
    # ms totals over 10 steps, one launch per step each
    phases = {"fwd_gemm": (3.2, 10), "bwd_dz_gemm": (3.4, 10), "bwd_dw_gemm": (4.7, 10), "bwd_dh_gemm": (3.2, 10),
              "target_scan": (0.42, 10), "fwd_combine": (0.16, 10)}
    r = bench._roofline(phases, cfg, steps, 1394.5, "measured", 6551.0, workload="llama")
    assert r["kernel"] == "bwd_dw_gemm" and r["bound"] == "hbm" and r["unit"] == "GB/s"
    # dW bytes per launch: fp32 V*d write + bf16 dZ^T + H reads
    byts = 4.0 * cfg.V * cfg.d + 2.0 * cfg.V * cfg.M + 2.0 * cfg.M * cfg.d
    assert abs(r["achieved"] - byts / 0.47e-3 / 1e9) <= 0.2
    assert abs(r["frac"] - r["achieved"] / 6551.0) <= 1e-3
    kinds = {p["kernel"]: p for p in r["phases"]}
    assert kinds["fwd_gemm"]["bound"] == "tensor"
    flops = 2.0 * cfg.M * cfg.V * cfg.d
    assert abs(kinds["fwd_gemm"]["achieved_tflops"] - flops / 0.32e-3 / 1e12) <= 0.2
    assert kinds["target_scan"]["bound"] == "hbm"          # G2 and G6 reported against HBM
    assert abs(kinds["target_scan"]["achieved_gbs"] - 2.0 * cfg.M * cfg.V / 0.042e-3 / 1e9) <= 0.2
    assert "fwd_combine" in kinds
    assert r["traffic"] is not None                          # committed capture of this workload
    r2 = bench._roofline(phases, cfg, steps, 1394.5, "measured", 6551.0, workload=None)
    assert r2["traffic"] is None


def test_roofline_tensor_bound_at_large_m(bench):
    import tracegen
    cfg = tracegen.CONFIGS["qwen3"]
    phases = {k: (15.0, 10) for k in ("fwd_gemm", "bwd_dz_gemm", "bwd_dh_gemm")}
    phases["bwd_dw_gemm"] = (16.5, 10)
    r = bench._roofline(phases, cfg, 10, 1394.5, "measured", 6551.0)
    assert r["kernel"] == "bwd_dw_gemm" and r["bound"] == "tensor" and r["unit"] == "TFLOP/s"


@pytest.mark.parametrize("name", ["ta_small", "ta_tiny"])
def test_tree_attn_work_counts_visible_pairs(bench, name):
    """bench._ta_work's algorithmic pair count equals the number of unmasked (row, key, head)
    triples of the oracle's mask (F4-R2), including ragged node counts and empty prefixes."""
    import numpy as np
    import tracegen
    from oracle import tree_attention as TA
    meta = tracegen.gen_tree_attn_meta(name)
    c = meta["cfg"]
    w = bench._ta_work(meta)
    off = meta["prefix_off"]
    pairs = 0
    for r in range(c.R):
        nn = c.N if meta["num_nodes"] is None else int(meta["num_nodes"][r])
        anc = TA.ancestor_rows(None if meta["parents"] is None else meta["parents"][r], nn, c.N)
        A = TA._allowed(anc, int(off[r + 1] - off[r]), c.N)
        pairs += int(A.sum())
    assert w["pairs"] == pairs * c.Hq
    assert w["fwd_flops"] == 4.0 * c.dh * w["pairs"] and w["bwd_flops"] == 10.0 * c.dh * w["pairs"]
    assert w["rows"] == c.R * (c.N + 1)
    kv = (int(np.diff(off).sum()) + c.R * (c.N + 1)) * c.Hkv * c.dh * 4
    assert w["fused_bytes"] >= 2 * kv                        # K/V read once + dK/dV written once

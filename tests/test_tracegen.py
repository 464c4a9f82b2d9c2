"""Trace generator contract (-m "not gpu"): determinism and structure."""
import numpy as np

import tracegen


def test_deterministic_and_shapes():
    a = tracegen.gen_trace("small")
    b = tracegen.gen_trace("small")
    for k in ("T_bits", "H_bits", "W_bits", "draft_tokens", "num_nodes"):
        np.testing.assert_array_equal(a[k], b[k])
    c = a["cfg"]
    assert a["T_bits"].shape == (c.M, c.V) and a["H_bits"].shape == (c.M, c.d)
    assert a["W_bits"].shape == (c.V, c.d) and a["draft_tokens"].shape == (c.R, c.N)
    assert a["draft_tokens"].min() >= 0 and a["draft_tokens"].max() < c.V


def test_tree_structure_and_distinct_siblings():
    t = tracegen.gen_trace("small_tree")
    P, X = t["parents"], t["draft_tokens"]
    R, N = X.shape
    for r in range(R):
        for n in range(N):
            assert -1 <= P[r, n] < n
        for p in set(P[r].tolist()):
            sib = X[r][P[r] == p]
            assert len(set(sib.tolist())) == len(sib)


def test_designated_token_is_strict_max():
    t = tracegen.gen_trace("small")
    T = tracegen.bf16_bits_to_f32(t["T_bits"])
    des = t["designated"]
    top = T[np.arange(T.shape[0]), des]
    T2 = T.copy()
    T2[np.arange(T.shape[0]), des] = -np.inf
    assert (top > T2.max(axis=1)).all()


def test_config_row_counts():
    assert tracegen.CONFIGS["llama"].M == 384
    assert tracegen.CONFIGS["qwen3"].M == 1792
    assert tracegen.CONFIGS["minimax"].M == 4608
    assert tracegen.CONFIGS["tree"].M == 25600
    assert tracegen.CONFIGS["tiny"].M == 20

"""ctypes binding of libaurora.so (include/aurora.h) — argument marshalling only.

Every step of the hot path runs inside the CUDA library; this module only turns
torch tensors (device memory, streams) into pointers and raises on non-OK status.
If libaurora.so is missing the import of the library fails loudly: there is no
CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AURORA_LIB") or os.path.join(_PKG, "libaurora.so")  # override: A/B experiments

AURORA_OK = 0
STATUS_NAMES = {0: "ok", 1: "invalid argument", 2: "structure", 3: "range", 4: "nonfinite", 5: "unsupported",
                6: "workspace", 7: "cuda", 8: "nccl"}
STATUS_NONFINITE, STATUS_RANGE, STATUS_STRUCTURE = 1, 2, 4
ROW_ACCEPT, ROW_DISCARD, ROW_PAD = 0, 1, 2
OP_VERIFY, OP_FWD, OP_BWD, OP_ALL = 0, 1, 2, 3
MAX_K, MAX_NODES = 16, 32

# Symbols declared in include/aurora.h (checked by tests/test_abi.py).
EXPORTS = ["aurora_workspace_size", "aurora_verify_labels", "aurora_spec_loss_fwd", "aurora_spec_loss_bwd",
           "aurora_comm_get_unique_id", "aurora_comm_create", "aurora_comm_create_loopback", "aurora_comm_destroy", "aurora_status_string",
           "aurora_build_info", "aurora_launch_count", "aurora_profile_enable", "aurora_profile_read",
           "aurora_debug_gemm", "aurora_debug_dlogits_rows", "aurora_set_option", "aurora_get_option",
           "aurora_verify_labels_topk", "aurora_adamw_workspace_size", "aurora_adamw_step",
           "aurora_profile_peek", "aurora_spec_loss_bwd_adamw", "aurora_tree_attn_fwd",
           "aurora_tree_attn_workspace_size", "aurora_tree_attn_bwd", "aurora_tree_rope",
           "aurora_draft_layer_workspace_size", "aurora_draft_layer_fwd", "aurora_draft_layer_bwd",
           "aurora_adamw_sharded_workspace_size", "aurora_adamw_step_sharded"]


class AuroraError(RuntimeError):
    def __init__(self, fn: str, status: int):
        self.status = status
        super().__init__(f"{fn} failed: {status} ({STATUS_NAMES.get(status, '?')})")


class aurora_trace_t(C.Structure):
    _fields_ = [("R", C.c_int32), ("N", C.c_int32), ("draft_tokens", C.c_void_p), ("parents", C.c_void_p),
                ("num_nodes", C.c_void_p), ("target_logits", C.c_void_p), ("ld_target", C.c_int64),
                ("V", C.c_int64), ("V_local", C.c_int64), ("vocab_offset", C.c_int64)]


class aurora_trace_topk_t(C.Structure):
    _fields_ = [("R", C.c_int32), ("N", C.c_int32), ("draft_tokens", C.c_void_p), ("parents", C.c_void_p),
                ("num_nodes", C.c_void_p), ("target_ids", C.c_void_p), ("target_vals", C.c_void_p),
                ("K_t", C.c_int32), ("V", C.c_int64)]


class aurora_loss_cfg_t(C.Structure):
    _fields_ = [("k_accept", C.c_int32), ("k_discard", C.c_int32), ("lambda_discard", C.c_float),
                ("normalize", C.c_int32), ("discard_scope", C.c_int32), ("accept_loss", C.c_int32),
                ("ntp_beta", C.c_float), ("discard_restricted", C.c_int32)]


class aurora_labels_t(C.Structure):
    _fields_ = [("k_max", C.c_int32), ("target_argmax", C.c_void_p), ("accepted", C.c_void_p),
                ("accept_len", C.c_void_p), ("bonus", C.c_void_p), ("row_class", C.c_void_p),
                ("sup_idx", C.c_void_p), ("sup_p", C.c_void_p), ("row_H", C.c_void_p), ("row_w", C.c_void_p),
                ("counts", C.c_void_p), ("status", C.c_void_p), ("row_lse_t", C.c_void_p), ("row_aux", C.c_void_p),
                ("target_logits", C.c_void_p), ("ld_target", C.c_int64), ("objective", C.c_int32),
                ("ntp_beta", C.c_float)]


class aurora_adamw_cfg_t(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("weight_decay", C.c_float), ("max_grad_norm", C.c_float), ("warmup_steps", C.c_int32)]


class aurora_tree_attn_t(C.Structure):
    _fields_ = [("R", C.c_int32), ("N", C.c_int32), ("Hq", C.c_int32), ("Hkv", C.c_int32), ("dh", C.c_int32),
                ("max_prefix", C.c_int32), ("prefix_total", C.c_int64), ("prefix_off", C.c_void_p), ("parents", C.c_void_p),
                ("num_nodes", C.c_void_p), ("scale", C.c_float), ("status", C.c_void_p)]


class aurora_draft_layer_t(C.Structure):
    _fields_ = [("ta", aurora_tree_attn_t), ("d", C.c_int32), ("I", C.c_int32), ("theta", C.c_float),
                ("eps", C.c_float)]


_DL_W = ["Wfc", "Wq", "Wk", "Wv", "Wo", "Wg", "Wu", "Wd", "we", "wh", "wpost", "wfinal"]


class aurora_draft_weights_t(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in _DL_W]


class aurora_draft_grads_t(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in _DL_W]


_lib = None


def lib() -> C.CDLL:
    """Load libaurora.so (in-tree).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} not found: build it with `python -m paper_2602_06932_b200.build` "
                           "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    vp, i64, i32, sz = C.c_void_p, C.c_int64, C.c_int32, C.c_size_t
    L.aurora_workspace_size.argtypes = [C.c_int, i64, i64, i64, C.POINTER(aurora_loss_cfg_t)]
    L.aurora_workspace_size.restype = sz
    L.aurora_verify_labels.argtypes = [C.POINTER(aurora_trace_t), C.POINTER(aurora_loss_cfg_t),
                                       C.POINTER(aurora_labels_t), vp, sz, vp, vp]
    L.aurora_verify_labels.restype = C.c_int
    L.aurora_spec_loss_fwd.argtypes = [vp, vp, i64, i64, i64, i64, C.POINTER(aurora_labels_t), vp, vp, vp, vp, sz,
                                       vp, vp]
    L.aurora_spec_loss_fwd.restype = C.c_int
    L.aurora_spec_loss_bwd.argtypes = [vp, vp, i64, i64, i64, i64, C.POINTER(aurora_labels_t), vp, vp, vp, vp,
                                       C.c_int, C.c_int, vp, sz, vp, vp]
    L.aurora_spec_loss_bwd.restype = C.c_int
    L.aurora_comm_get_unique_id.argtypes = [vp]
    L.aurora_comm_get_unique_id.restype = C.c_int
    L.aurora_comm_create.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
    L.aurora_comm_create.restype = C.c_int
    L.aurora_comm_destroy.argtypes = [vp]
    L.aurora_comm_create_loopback.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
    L.aurora_comm_create_loopback.restype = C.c_int
    L.aurora_comm_destroy.restype = C.c_int
    L.aurora_status_string.argtypes = [C.c_int]
    L.aurora_status_string.restype = C.c_char_p
    L.aurora_build_info.argtypes = []
    L.aurora_build_info.restype = C.c_char_p
    L.aurora_launch_count.argtypes = []
    L.aurora_launch_count.restype = C.c_uint64
    L.aurora_profile_enable.argtypes = [C.c_int]
    L.aurora_profile_enable.restype = None
    L.aurora_profile_read.argtypes = [C.POINTER(C.c_char_p), C.POINTER(C.c_float), C.POINTER(C.c_int32), C.c_int]
    L.aurora_profile_read.restype = C.c_int
    L.aurora_profile_peek.argtypes = [C.POINTER(C.c_char_p), C.POINTER(C.c_float), C.POINTER(C.c_int32), C.c_int]
    L.aurora_profile_peek.restype = C.c_int
    L.aurora_debug_gemm.argtypes = [C.c_int, C.c_int, vp, vp, vp, i64, i64, i64, i64, i64, i64, vp]
    L.aurora_debug_gemm.restype = C.c_int
    L.aurora_debug_dlogits_rows.argtypes = [vp, vp, i64, i64, i64, i64, C.POINTER(aurora_labels_t), vp, vp, vp,
                                            i32, vp, vp]
    L.aurora_debug_dlogits_rows.restype = C.c_int
    L.aurora_verify_labels_topk.argtypes = [C.POINTER(aurora_trace_topk_t), C.POINTER(aurora_loss_cfg_t),
                                            C.POINTER(aurora_labels_t), vp, sz, vp, vp]
    L.aurora_verify_labels_topk.restype = C.c_int
    L.aurora_set_option.argtypes = [C.c_char_p, C.c_int64]
    L.aurora_spec_loss_bwd_adamw.argtypes = [vp, vp, i64, i64, i64, i64, C.POINTER(aurora_labels_t), vp, vp, vp, vp,
                                             vp, vp, i64, C.POINTER(aurora_adamw_cfg_t), vp, vp, vp, sz, vp, sz, vp,
                                             vp]
    L.aurora_adamw_workspace_size.argtypes = [i64]
    L.aurora_adamw_workspace_size.restype = sz
    L.aurora_adamw_step.argtypes = [vp, vp, vp, vp, vp, i64, i64, C.POINTER(aurora_adamw_cfg_t), vp, vp, vp, sz, vp,
                                    vp]
    L.aurora_set_option.restype = C.c_int
    L.aurora_adamw_sharded_workspace_size.argtypes = [i64, C.c_int]
    L.aurora_adamw_sharded_workspace_size.restype = sz
    L.aurora_adamw_step_sharded.argtypes = [vp, vp, vp, vp, vp, i64, i64, C.POINTER(aurora_adamw_cfg_t), vp, vp, vp,
                                            sz, vp, vp]
    L.aurora_adamw_step_sharded.restype = C.c_int
    L.aurora_tree_attn_fwd.argtypes = [C.POINTER(aurora_tree_attn_t), vp, vp, vp, vp, vp, vp, vp, vp]
    L.aurora_tree_attn_fwd.restype = C.c_int
    L.aurora_tree_attn_workspace_size.argtypes = [C.POINTER(aurora_tree_attn_t)]
    L.aurora_tree_attn_workspace_size.restype = sz
    L.aurora_tree_attn_bwd.argtypes = [C.POINTER(aurora_tree_attn_t)] + [vp] * 14 + [sz, vp]
    L.aurora_tree_attn_bwd.restype = C.c_int
    L.aurora_tree_rope.argtypes = [C.POINTER(aurora_tree_attn_t), vp, C.c_int, vp, C.c_int, C.c_float, C.c_int, vp]
    L.aurora_tree_rope.restype = C.c_int
    L.aurora_draft_layer_workspace_size.argtypes = [C.POINTER(aurora_draft_layer_t)]
    L.aurora_draft_layer_workspace_size.restype = sz
    L.aurora_draft_layer_fwd.argtypes = [C.POINTER(aurora_draft_layer_t), C.POINTER(aurora_draft_weights_t)] + \
        [vp] * 6 + [sz, vp]
    L.aurora_draft_layer_fwd.restype = C.c_int
    L.aurora_draft_layer_bwd.argtypes = [C.POINTER(aurora_draft_layer_t), C.POINTER(aurora_draft_weights_t)] + \
        [vp] * 5 + [C.POINTER(aurora_draft_grads_t)] + [vp] * 5 + [sz, vp]
    L.aurora_draft_layer_bwd.restype = C.c_int
    L.aurora_get_option.argtypes = [C.c_char_p]
    L.aurora_get_option.restype = C.c_int64
    _lib = L
    return L


def _check(fn: str, st: int):
    if st != AURORA_OK:
        raise AuroraError(fn, st)


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _expect(t, dtype_name: str, what: str):
    """Marshalling-level check: the C-ABI cannot see dtypes, so a wrong one would be
    silently reinterpreted.  Raises before anything is enqueued."""
    if t is None:
        return
    import torch
    want = {"bf16": torch.bfloat16, "f32": torch.float32, "i32": torch.int32, "u8": torch.uint8}[dtype_name]
    if t.dtype != want:
        raise TypeError(f"{what}: expected {want}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{what}: must be contiguous")


def torch_f32():
    import torch
    return torch.float32


def _stream(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


# ----------------------------------------------------------- thin C-name wrappers
def aurora_workspace_size(op: int, M: int, d: int, V_local: int, cfg: aurora_loss_cfg_t) -> int:
    return int(lib().aurora_workspace_size(op, M, d, V_local, C.byref(cfg)))


def aurora_verify_labels(trace: aurora_trace_t, cfg: aurora_loss_cfg_t, labels: aurora_labels_t, ws, ws_bytes: int,
                         comm=None, stream=None) -> None:
    _check("aurora_verify_labels", lib().aurora_verify_labels(C.byref(trace), C.byref(cfg), C.byref(labels),
                                                              ws, ws_bytes, comm, _stream(stream)))


def aurora_spec_loss_fwd(H, W, M, d, V_local, vocab_offset, labels, row_lse, row_loss, loss, ws, ws_bytes,
                         comm=None, stream=None) -> None:
    _expect(H, "bf16", "H"); _expect(W, "bf16", "W")
    _expect(row_lse, "f32", "row_lse"); _expect(row_loss, "f32", "row_loss"); _expect(loss, "f32", "loss")
    _check("aurora_spec_loss_fwd", lib().aurora_spec_loss_fwd(
        _ptr(H), _ptr(W), M, d, V_local, vocab_offset, C.byref(labels), _ptr(row_lse), _ptr(row_loss), _ptr(loss),
        ws, ws_bytes, comm, _stream(stream)))


def aurora_spec_loss_bwd(H, W, M, d, V_local, vocab_offset, labels, row_lse, dloss, dH, dW, dW_is_bf16,
                         accumulate_dW, ws, ws_bytes, comm=None, stream=None) -> None:
    _expect(H, "bf16", "H"); _expect(W, "bf16", "W"); _expect(row_lse, "f32", "row_lse")
    _expect(dloss, "f32", "dloss"); _expect(dH, "f32", "dH"); _expect(dW, "bf16" if dW_is_bf16 else "f32", "dW")
    _check("aurora_spec_loss_bwd", lib().aurora_spec_loss_bwd(
        _ptr(H), _ptr(W), M, d, V_local, vocab_offset, C.byref(labels), _ptr(row_lse), _ptr(dloss), _ptr(dH),
        _ptr(dW), int(dW_is_bf16), int(accumulate_dW), ws, ws_bytes, comm, _stream(stream)))


def aurora_debug_gemm(a_mn: bool, b_mn: bool, A, B, D, M, N, K, lda, ldb, ldd, stream=None) -> None:
    _expect(A, "bf16", "A"); _expect(B, "bf16", "B"); _expect(D, "f32", "D")
    _check("aurora_debug_gemm", lib().aurora_debug_gemm(int(a_mn), int(b_mn), _ptr(A), _ptr(B), _ptr(D), M, N, K,
                                                        lda, ldb, ldd, _stream(stream)))


def aurora_adamw_step(W_master, W_bf16, m, v, dW, step: int, cfg: aurora_adamw_cfg_t, ws, extra_sq=None,
                      grad_norm=None, comm=None, stream=None) -> None:
    """NEXT F3: one fused AdamW step (global-norm clip, warm-up LR) on fp32 master weights.
    step >= 1, or 0 = the device step counter kept in `ws` (graph-replay safe)."""
    for t, n in ((W_master, "W_master"), (m, "m"), (v, "v"), (dW, "dW")):
        _expect(t, "f32", n)
    _expect(W_bf16, "bf16", "W_bf16")
    _check("aurora_adamw_step", lib().aurora_adamw_step(
        _ptr(W_master), _ptr(W_bf16), _ptr(m), _ptr(v), _ptr(dW), W_master.numel(), int(step), C.byref(cfg),
        _ptr(extra_sq), _ptr(grad_norm), _ptr(ws), ws.numel() if ws is not None else 0, comm, _stream(stream)))


class AdamW:
    """Owns the fp32 moments and workspace of a fused AdamW over one fp32 master tensor
    (defaults: P:487-489 / Table 3 — lr 1e-5, wd 0.0, clip 0.5, 400 warm-up steps;
    betas / eps per SPEC's design decision).  The step counter lives on the device (in the
    zero-initialised workspace), so a captured CUDA graph advances it on every replay;
    `step_count` mirrors it on the host for eager use."""

    def __init__(self, W_master, lr: float = 1e-5, betas=(0.9, 0.999), eps: float = 1e-8, weight_decay: float = 0.0,
                 max_grad_norm: float = 0.5, warmup_steps: int = 400, comm=None):
        import torch
        self.W = W_master
        self.m = torch.zeros_like(W_master)
        self.v = torch.zeros_like(W_master)
        self.cfg = aurora_adamw_cfg_t(lr, betas[0], betas[1], eps, weight_decay, max_grad_norm, warmup_steps)
        n = int(lib().aurora_adamw_workspace_size(W_master.numel()))
        self.ws = torch.zeros(n, dtype=torch.uint8, device=W_master.device)
        self.grad_norm = torch.zeros(1, dtype=torch.float32, device=W_master.device)
        self.step_count = 0
        self.comm = comm

    def step(self, dW, W_bf16=None, extra_sq=None, stream=None):
        self.step_count += 1
        aurora_adamw_step(self.W, W_bf16, self.m, self.v, dW, 0, self.cfg, self.ws, extra_sq,
                          self.grad_norm, self.comm, stream)


class ShardedAdamW:
    """F3 under data parallelism (aurora_adamw_step_sharded): this DP rank owns shard
    `dp_rank` of the fp32 master / moments of a flat lm_head of n elements; each step
    reduce-scatters the (unreduced) dW over the DP group, updates the shard and allgathers
    the bf16 weights every rank's GEMMs read."""

    def __init__(self, W_master_full, comm, dp_rank: int, dp_size: int, lr: float = 1e-5, betas=(0.9, 0.999),
                 eps: float = 1e-8, weight_decay: float = 0.0, max_grad_norm: float = 0.5, warmup_steps: int = 400):
        import torch
        n = W_master_full.numel()
        if n % (4 * dp_size):
            raise ValueError("n must be a multiple of 4 * dp_size")
        sh = n // dp_size
        self.n, self.comm = n, comm
        self.W = W_master_full.reshape(-1)[dp_rank * sh:(dp_rank + 1) * sh].clone()
        self.m = torch.zeros_like(self.W)
        self.v = torch.zeros_like(self.W)
        self.cfg = aurora_adamw_cfg_t(lr, betas[0], betas[1], eps, weight_decay, max_grad_norm, warmup_steps)
        nb = int(lib().aurora_adamw_sharded_workspace_size(n, dp_size))
        self.ws = torch.zeros(nb, dtype=torch.uint8, device=self.W.device)
        self.grad_norm = torch.zeros(1, dtype=torch.float32, device=self.W.device)

    def step(self, dW, W_bf16, extra_sq=None, stream=None):
        _expect(dW, "f32", "dW")
        _expect(W_bf16, "bf16", "W_bf16")
        _check("aurora_adamw_step_sharded", lib().aurora_adamw_step_sharded(
            _ptr(self.W), _ptr(W_bf16), _ptr(self.m), _ptr(self.v), _ptr(dW), self.n, 0, C.byref(self.cfg),
            _ptr(extra_sq), _ptr(self.grad_norm), _ptr(self.ws), self.ws.numel(), self.comm, _stream(stream)))


def aurora_set_option(name: str, value: int) -> None:
    _check("aurora_set_option", lib().aurora_set_option(name.encode(), int(value)))


def aurora_get_option(name: str) -> int:
    return int(lib().aurora_get_option(name.encode()))


def aurora_launch_count() -> int:
    return int(lib().aurora_launch_count())


def aurora_build_info() -> str:
    return lib().aurora_build_info().decode()


def aurora_profile_enable(on: bool) -> None:
    lib().aurora_profile_enable(1 if on else 0)


def aurora_profile_read(peek: bool = False) -> dict:
    """Per-phase (total ms, launches) since the last read; peek=True keeps the events (a
    captured CUDA graph re-times them on every replay)."""
    n = 32
    names = (C.c_char_p * n)()
    ms = (C.c_float * n)()
    cnt = (C.c_int32 * n)()
    fn = lib().aurora_profile_peek if peek else lib().aurora_profile_read
    k = fn(names, ms, cnt, n)
    return {names[i].decode(): (float(ms[i]), int(cnt[i])) for i in range(k)}


def aurora_comm_get_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check("aurora_comm_get_unique_id", lib().aurora_comm_get_unique_id(buf))
    return buf.raw


def aurora_comm_create(uid: bytes, nranks: int, rank: int, vp_size: int, dp_size: int):
    h = C.c_void_p()
    buf = C.create_string_buffer(uid, 128)
    _check("aurora_comm_create", lib().aurora_comm_create(buf, nranks, rank, vp_size, dp_size, C.byref(h)))
    return h


def aurora_comm_create_loopback(nranks: int, vp_size: int, dp_size: int) -> list:
    """`nranks` virtual-rank communicators on the current device (one host thread + stream
    per rank; see include/aurora.h)."""
    hs = (C.c_void_p * nranks)()
    _check("aurora_comm_create_loopback", lib().aurora_comm_create_loopback(nranks, vp_size, dp_size, hs))
    return [C.c_void_p(h) for h in hs]


def aurora_comm_destroy(h) -> None:
    _check("aurora_comm_destroy", lib().aurora_comm_destroy(h))


# ----------------------------------------------------------- public step API
class SpecTrainStep:
    """Owns the label buffers and workspace for one trace-batch shape and runs
    verify -> fwd -> bwd through the C-ABI on the current CUDA stream.

    Shapes: R requests x N nodes (M = R(N+1) rows), hidden d, global vocab V, this
    rank's vocab slice [vocab_offset, vocab_offset + V_local).
    """

    def __init__(self, R: int, N: int, d: int, V: int, V_local: Optional[int] = None, vocab_offset: int = 0,
                 k_accept: int = 1, k_discard: int = 10, lambda_discard: float = 1.0, normalize: int = 0,
                 discard_scope: int = 0, device="cuda", comm=None, accept_loss: str = "fkl", ntp_beta: float = 0.0,
                 discard_loss: str = "full"):
        import torch
        self.R, self.N, self.d, self.V = R, N, d, V
        self.V_local = V if V_local is None else V_local
        self.vocab_offset = vocab_offset
        self.M = R * (N + 1)
        self.comm = comm
        if accept_loss not in ("fkl", "rkl"):
            raise ValueError("accept_loss must be 'fkl' or 'rkl'")
        if discard_loss not in ("full", "restricted"):
            raise ValueError("discard_loss must be 'full' or 'restricted'")
        self.cfg = aurora_loss_cfg_t(k_accept, k_discard, lambda_discard, normalize, discard_scope,
                                     1 if accept_loss == "rkl" else 0, ntp_beta,
                                     1 if discard_loss == "restricted" else 0)
        self.k_max = max(k_accept, k_discard, 1)
        dev = torch.device(device)
        M, km = self.M, self.k_max
        i32, u8, f32 = torch.int32, torch.uint8, torch.float32
        self.target_argmax = torch.empty(M, dtype=i32, device=dev)
        self.accepted = torch.empty(R, N, dtype=u8, device=dev)
        self.accept_len = torch.empty(R, dtype=i32, device=dev)
        self.bonus = torch.empty(R, dtype=i32, device=dev)
        self.row_class = torch.empty(M, dtype=u8, device=dev)
        self.sup_idx = torch.empty(M, km, dtype=i32, device=dev)
        self.sup_p = torch.empty(M, km, dtype=f32, device=dev)
        self.row_H = torch.empty(M, dtype=f32, device=dev)
        self.row_w = torch.empty(M, dtype=f32, device=dev)
        self.counts = torch.empty(2, dtype=i32, device=dev)
        self.status = torch.zeros(1, dtype=i32, device=dev)
        self.row_lse = torch.empty(M, dtype=f32, device=dev)
        self.row_loss = torch.empty(M, dtype=f32, device=dev)
        self.loss = torch.empty(1, dtype=f32, device=dev)
        self.row_lse_t = torch.empty(M, dtype=f32, device=dev)
        self.row_aux = torch.empty(M, dtype=f32, device=dev)
        self.labels = aurora_labels_t(km, *(t.data_ptr() for t in (
            self.target_argmax, self.accepted, self.accept_len, self.bonus, self.row_class, self.sup_idx,
            self.sup_p, self.row_H, self.row_w, self.counts, self.status, self.row_lse_t, self.row_aux)), None, 0, 0,
            0.0)
        self._target_ref = None
        self.ws_bytes = aurora_workspace_size(OP_ALL, M, d, self.V_local, self.cfg)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)

    def verify(self, draft_tokens, target_logits, parents=None, num_nodes=None, stream=None):
        _expect(draft_tokens, "i32", "draft_tokens"); _expect(parents, "i32", "parents")
        _expect(num_nodes, "i32", "num_nodes"); _expect(target_logits, "bf16", "target_logits")
        t = aurora_trace_t(self.R, self.N, _ptr(draft_tokens), _ptr(parents), _ptr(num_nodes), _ptr(target_logits),
                           target_logits.stride(0), self.V, self.V_local, self.vocab_offset)
        # F2 objectives read T again in fwd / bwd: the labels reference it (kept alive here)
        self.labels.target_logits = _ptr(target_logits)
        self.labels.ld_target = target_logits.stride(0)
        self._target_ref = target_logits
        aurora_verify_labels(t, self.cfg, self.labels, self.ws.data_ptr(), self.ws_bytes, self.comm, stream)

    def verify_topk(self, draft_tokens, target_ids, target_vals, parents=None, num_nodes=None, stream=None):
        """NEXT F1: labels from the transmitted top-K target payload (ids int32 [M, K_t],
        bf16 logits [M, K_t]) instead of dense logits."""
        _expect(draft_tokens, "i32", "draft_tokens"); _expect(parents, "i32", "parents")
        _expect(num_nodes, "i32", "num_nodes"); _expect(target_ids, "i32", "target_ids")
        _expect(target_vals, "bf16", "target_vals")
        K_t = target_ids.shape[1]
        need = aurora_workspace_size(OP_VERIFY, self.M, self.d, K_t, self.cfg)
        if need > self.ws_bytes:
            raise ValueError("workspace too small for this K_t")
        t = aurora_trace_topk_t(self.R, self.N, _ptr(draft_tokens), _ptr(parents), _ptr(num_nodes), _ptr(target_ids),
                                _ptr(target_vals), K_t, self.V)
        self.labels.target_logits = None
        self.labels.ld_target = 0
        self._target_ref = None
        _check("aurora_verify_labels_topk", lib().aurora_verify_labels_topk(
            C.byref(t), C.byref(self.cfg), C.byref(self.labels), self.ws.data_ptr(), self.ws_bytes, self.comm,
            _stream(stream)))

    def forward(self, H, W, stream=None):
        aurora_spec_loss_fwd(H, W, self.M, self.d, self.V_local, self.vocab_offset, self.labels, self.row_lse,
                             self.row_loss, self.loss, self.ws.data_ptr(), self.ws_bytes, self.comm, stream)
        return self.loss

    def backward(self, H, W, dH, dW, dloss=None, accumulate_dW=False, stream=None, dp_reduce=True):
        """dW: fp32 or bf16 [V_local, d].  dp_reduce=False: leave dW unreduced over the
        DP group (ShardedAdamW reduce-scatters it)."""
        flags = (1 if accumulate_dW else 0) | (0 if dp_reduce else 2)
        aurora_spec_loss_bwd(H, W, self.M, self.d, self.V_local, self.vocab_offset, self.labels, self.row_lse,
                             dloss, dH, dW, dW.dtype != torch_f32(), flags, self.ws.data_ptr(), self.ws_bytes,
                             self.comm, stream)

    def backward_adamw(self, H, W, dH, opt: "AdamW", dloss=None, extra_sq=None, stream=None):
        """NEXT F3 fused: backward (dH) + the AdamW step applied from the dW GEMM epilogue
        (dW never materialised).  opt owns the fp32 master of W, its moments and workspace;
        W (bf16) is rewritten from the updated master."""
        _expect(H, "bf16", "H"); _expect(W, "bf16", "W"); _expect(dH, "f32", "dH")
        opt.step_count += 1
        _check("aurora_spec_loss_bwd_adamw", lib().aurora_spec_loss_bwd_adamw(
            _ptr(H), _ptr(W), self.M, self.d, self.V_local, self.vocab_offset, C.byref(self.labels), _ptr(self.row_lse),
            _ptr(dloss), _ptr(dH), _ptr(opt.W), _ptr(opt.m), _ptr(opt.v), 0, C.byref(opt.cfg),
            _ptr(extra_sq), _ptr(opt.grad_norm), _ptr(self.ws), self.ws_bytes, _ptr(opt.ws), opt.ws.numel(),
            self.comm, _stream(stream)))
    def step(self, draft_tokens, target_logits, H, W, dH, dW, parents=None, num_nodes=None, stream=None):
        self.verify(draft_tokens, target_logits, parents, num_nodes, stream)
        self.forward(H, W, stream)
        self.backward(H, W, dH, dW, stream=stream)
        return self.loss

    def debug_dlogits_rows(self, H, W, rows, dloss=None, stream=None):
        import torch
        out = torch.empty(len(rows), self.V_local, dtype=torch.float32, device=H.device)
        r = torch.as_tensor(rows, dtype=torch.int32, device=H.device)
        _check("aurora_debug_dlogits_rows", lib().aurora_debug_dlogits_rows(
            _ptr(H), _ptr(W), self.M, self.d, self.V_local, self.vocab_offset, C.byref(self.labels),
            _ptr(self.row_lse), _ptr(dloss), _ptr(r), len(rows), _ptr(out), _stream(stream)))
        return out


# ----------------------------------------------------------------------------- NEXT F4
class TreeAttention:
    """Tree attention of the draft layer (include/aurora.h aurora_tree_attn_*).

    Marshalling only: holds the batch structure (prefix offsets, parents, node counts, all
    device int32) and the device status word / backward workspace, and calls the library.
    Q/O/dO bf16 [R, N+1, Hq, dh]; Kt/Vt bf16 [R, N+1, Hkv, dh]; Kp/Vp bf16 [P_total, Hkv, dh];
    lse f32 [R, N+1, Hq]; dQ f32 like Q; dK*/dV* bf16 like their inputs."""

    def __init__(self, R: int, N: int, Hq: int, Hkv: int, dh: int, prefix_off, max_prefix: int,
                 parents=None, num_nodes=None, scale: float = 0.0, device=None, prefix_total: int = None):
        import torch
        dev = device or prefix_off.device
        _expect(prefix_off, "i32", "prefix_off")
        _expect(parents, "i32", "parents")
        _expect(num_nodes, "i32", "num_nodes")
        self.R, self.N, self.Hq, self.Hkv, self.dh = R, N, Hq, Hkv, dh
        self.prefix_off, self.parents, self.num_nodes = prefix_off, parents, num_nodes
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        if prefix_total is None:   # one small D2H read at construction, not per call
            prefix_total = int(prefix_off[-1].item())
        self.cfg = aurora_tree_attn_t(R, N, Hq, Hkv, dh, int(max_prefix), int(prefix_total), _ptr(prefix_off),
                                      _ptr(parents),
                                      _ptr(num_nodes), float(scale), _ptr(self.status))
        nbytes = int(lib().aurora_tree_attn_workspace_size(C.byref(self.cfg)))
        self.ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)

    def forward(self, Q, Kt, Vt, Kp, Vp, O, lse, stream=None):
        for t, n in [(Q, "Q"), (Kt, "Kt"), (Vt, "Vt"), (Kp, "Kp"), (Vp, "Vp"), (O, "O")]:
            _expect(t, "bf16", n)
        _expect(lse, "f32", "lse")
        _check("aurora_tree_attn_fwd", lib().aurora_tree_attn_fwd(
            C.byref(self.cfg), _ptr(Q), _ptr(Kt), _ptr(Vt), _ptr(Kp), _ptr(Vp), _ptr(O), _ptr(lse),
            _stream(stream)))

    def backward(self, Q, Kt, Vt, Kp, Vp, O, lse, dO, dQ, dKt, dVt, dKp, dVp, stream=None):
        for t, n in [(Q, "Q"), (Kt, "Kt"), (Vt, "Vt"), (Kp, "Kp"), (Vp, "Vp"), (O, "O"), (dO, "dO"),
                     (dKt, "dKt"), (dVt, "dVt"), (dKp, "dKp"), (dVp, "dVp")]:
            _expect(t, "bf16", n)
        _expect(lse, "f32", "lse")
        _expect(dQ, "f32", "dQ")
        _check("aurora_tree_attn_bwd", lib().aurora_tree_attn_bwd(
            C.byref(self.cfg), _ptr(Q), _ptr(Kt), _ptr(Vt), _ptr(Kp), _ptr(Vp), _ptr(O), _ptr(lse), _ptr(dO),
            _ptr(dQ), _ptr(dKt), _ptr(dVt), _ptr(dKp), _ptr(dVp), _ptr(self.ws), self.ws.numel(),
            _stream(stream)))

    def rope(self, Q=None, Kt=None, theta: float = 500000.0, inverse: bool = False, stream=None):
        """In-place tree-position RoPE of Q and/or the tree keys Kt (bf16 or f32 tensors)."""
        for t, n in [(Q, "Q"), (Kt, "Kt")]:
            if t is not None:
                _expect(t, "f32" if t.dtype.is_floating_point and t.element_size() == 4 else "bf16", n)
        q32 = int(Q is not None and Q.element_size() == 4)
        k32 = int(Kt is not None and Kt.element_size() == 4)
        _check("aurora_tree_rope", lib().aurora_tree_rope(C.byref(self.cfg), _ptr(Q), q32, _ptr(Kt), k32,
                                                          float(theta), int(bool(inverse)), _stream(stream)))


class DraftLayer:
    """F4 draft layer (include/aurora.h aurora_draft_layer_*, reading F4-R7): marshalling only.
    `ta` is a TreeAttention (batch structure + heads); W maps the names of aurora_draft_weights_t
    to device tensors (bf16 matrices, f32 norm weights)."""

    def __init__(self, ta: "TreeAttention", d: int, I: int, W: dict, theta: float = 500000.0, eps: float = 1e-6):
        import torch
        for n in _DL_W:
            _expect(W[n], "f32" if n in ("we", "wh", "wpost", "wfinal") else "bf16", n)
        self.ta, self.W = ta, W
        self.cfg = aurora_draft_layer_t(ta.cfg, d, I, float(theta), float(eps))
        self.w = aurora_draft_weights_t(*[_ptr(W[n]) for n in _DL_W])
        nbytes = int(lib().aurora_draft_layer_workspace_size(C.byref(self.cfg)))
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=ta.status.device)

    def forward(self, h3, e, Kp, Vp, H, stream=None):
        for t, n in [(h3, "h3"), (e, "e"), (Kp, "Kp"), (Vp, "Vp"), (H, "H")]:
            _expect(t, "bf16", n)
        _check("aurora_draft_layer_fwd", lib().aurora_draft_layer_fwd(
            C.byref(self.cfg), C.byref(self.w), _ptr(h3), _ptr(e), _ptr(Kp), _ptr(Vp), _ptr(H), _ptr(self.ws),
            self.ws.numel(), _stream(stream)))

    def backward(self, h3, e, Kp, Vp, dH, G: dict, dh3, de, dKp, dVp, stream=None):
        _expect(dH, "f32", "dH")
        for n in _DL_W:
            _expect(G[n], "f32", "G." + n)
        g = aurora_draft_grads_t(*[_ptr(G[n]) for n in _DL_W])
        _check("aurora_draft_layer_bwd", lib().aurora_draft_layer_bwd(
            C.byref(self.cfg), C.byref(self.w), _ptr(h3), _ptr(e), _ptr(Kp), _ptr(Vp), _ptr(dH), C.byref(g),
            _ptr(dh3), _ptr(de), _ptr(dKp), _ptr(dVp), _ptr(self.ws), self.ws.numel(), _stream(stream)))


class SpeculatorStep:
    """One whole speculator training step (marshalling only; every stage is a library call on
    the current stream): greedy verification + labels (A2-A4) -> draft layer forward (F4) -> H
    -> lm_head forward / backward with the Eq. 3 loss (A5-A9) -> dH -> draft layer backward (F4).
    `spec` (SpecTrainStep) and `layer` (DraftLayer) must describe the same batch (R, N, tree)."""

    def __init__(self, spec: "SpecTrainStep", layer: "DraftLayer"):
        if spec.R != layer.ta.R or spec.N != layer.ta.N or spec.d != layer.cfg.d:
            raise ValueError("SpeculatorStep: spec and layer shapes differ")
        self.spec, self.layer = spec, layer

    def step(self, draft_tokens, T, h3, e, Kp, Vp, W_lm, H, dH, dW_lm, G, dh3, de, dKp, dVp, parents=None,
             num_nodes=None, stream=None):
        """The tree (parents, ragged node counts) is the layer's TreeAttention's: verification,
        the tree-attention mask, tree RoPE and the prefix layout all follow the same batch.
        `parents` / `num_nodes`, if given, must be those very tensors (a different tree would
        silently mix two batches)."""
        ta = self.layer.ta
        for given, own, name in ((parents, ta.parents, "parents"), (num_nodes, ta.num_nodes, "num_nodes")):
            if given is not None and (own is None or given.data_ptr() != own.data_ptr() or given.shape != own.shape):
                raise ValueError(f"SpeculatorStep.step: {name} differs from the layer's TreeAttention {name}; "
                                 "build a TreeAttention / DraftLayer for the new batch")
        self.spec.verify(draft_tokens, T, ta.parents, ta.num_nodes, stream)
        self.layer.forward(h3, e, Kp, Vp, H, stream)
        self.spec.forward(H, W_lm, stream)
        self.spec.backward(H, W_lm, dH, dW_lm, stream=stream)
        self.layer.backward(h3, e, Kp, Vp, dH, G, dh3, de, dKp, dVp, stream)
        return self.spec.loss


class SpeculatorParams:
    """Every trainable speculator parameter (the F4 draft layer's and the lm_head W) in three flat
    device buffers — fp32 master, the bf16 copy the GEMMs read, fp32 gradients — so that ONE
    aurora_adamw_step (F3) updates all of them under one global gradient norm (clip 0.5
    over the model).  `W` / `G` are views into the buffers (the norm weights' views are fp32 slices
    of the master: the kernels read them directly); `W_lm` / `dW_lm` are the lm_head's."""

    NORMS = ("we", "wh", "wpost", "wfinal")

    def __init__(self, d: int, I: int, Hq: int, Hkv: int, dh: int, V: int, device):
        import torch
        qd, kd = Hq * dh, Hkv * dh
        self.shapes = [("W_lm", (V, d)), ("Wfc", (d, 3 * d)), ("Wq", (qd, 2 * d)), ("Wk", (kd, 2 * d)),
                       ("Wv", (kd, 2 * d)), ("Wo", (d, qd)), ("Wg", (I, d)), ("Wu", (I, d)), ("Wd", (d, I)),
                       ("we", (d,)), ("wh", (d,)), ("wpost", (d,)), ("wfinal", (d,))]
        sizes = [int(np.prod(s)) for _, s in self.shapes]
        total = int(sum(sizes))
        self.master = torch.zeros(total, dtype=torch.float32, device=device)
        self.bf = torch.zeros(total, dtype=torch.bfloat16, device=device)
        self.grad = torch.zeros(total, dtype=torch.float32, device=device)
        self.W, self.G, self.M, o = {}, {}, {}, 0
        for (name, shape), n in zip(self.shapes, sizes):
            self.M[name] = self.master[o:o + n].view(shape)
            self.W[name] = self.M[name] if name in self.NORMS else self.bf[o:o + n].view(shape)
            self.G[name] = self.grad[o:o + n].view(shape)
            o += n
        self.W_lm, self.dW_lm = self.W.pop("W_lm"), self.G.pop("W_lm")

    def load(self, values: dict):
        """Set the fp32 master from host / device arrays by name and refresh the bf16 copy."""
        import torch
        for name, v in values.items():
            self.M[name].copy_(torch.as_tensor(np.asarray(v, np.float32)))
        self.bf.copy_(self.master.to(torch.bfloat16))

    def adamw(self, **kw) -> "AdamW":
        """One AdamW over every speculator parameter.  Single-rank only: under vocab
        parallelism the flat buffer mixes the sharded lm_head with draft-layer parameters
        replicated on every rank, whose squares a VP norm allreduce would count vp_size
        times."""
        if kw.get("comm") is not None:
            raise ValueError("SpeculatorParams.adamw is single-rank (replicated draft-layer gradients would be "
                             "counted once per VP rank in the global norm)")
        return AdamW(self.master, **kw)

    def optimizer_step(self, opt: "AdamW", stream=None):
        opt.step(self.grad, W_bf16=self.bf, stream=stream)

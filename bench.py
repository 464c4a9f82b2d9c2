#!/usr/bin/env python
"""Bench: speculator-training tokens/s of the Aurora hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama] [--impl ours|reference]

A step = one pass of the whole hot path over one synthetic
trace batch: greedy verification + labels, lm_head fwd with vocab-wide
log-softmax + Eq. 3 loss, and the bwd (dLogits tiles -> dW, dH).  Inputs are
resident in HBM when the timed region starts; every step is bracketed by its own
CUDA events on the launching stream, L2 is flushed between steps (a 256 MiB write,
outside the events).  `value` = rows (training tokens) processed by all ranks /
max-over-ranks time.  `e2e` repeats the measurement through the public API with the
trace batch (T, H, draft tokens) copied from pinned host memory every step and the
loss + accept lengths read back.

Default workload: `qwen3` (BASELINE.json configs[2], the largest configuration that fits
one GPU; configs[1] `llama` and the others via --config).

N > 1 (torchrun): vocab-parallel lm_head by default (weak scaling: one global batch of
N x R requests, rank p owns vocab slice p of W and T; C1/C3 per-row exchanges and the C4
dH allreduce); `--vp A --dp B` (A x B = N) is the 2-D DP x VP layout; `--parallel dp` is
pure data parallelism (C2 counts + C5 dW allreduce).

--impl reference: the f64 CPU oracle (the reference arm for this tier) timed on the
host cores on a bounded sample of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import tracegen  # noqa: E402


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("bf16_tflops", 1624.6), d.get("bf16_tflops_sustained", 1394.5), d.get("hbm_gbs", 6551.0), "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML polled every 2 ms
    from a thread (a graph-replayed timed region lasts only tens of ms), else nvidia-smi
    -lms 100.  Reasons: hw_slowdown, hw_thermal_slowdown, sw_thermal_slowdown, sw_power_cap."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NVML_BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, gpu_index: int):
        idx = gpu_index
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                idx = int(vis.split(",")[gpu_index])
            except (ValueError, IndexError):
                idx = gpu_index
        self.idx = idx
        self.rows = []      # nvidia-smi rows
        self.sm, self.mx, self.reasons = [], [], set()
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self.mx.append(float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)))
            self._sample_nvml()  # one sample at the start of the timed region
            self.t = threading.Thread(target=self._poll_nvml, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _sample_nvml(self):
        n = self.nvml
        self.sm.append(float(n.nvmlDeviceGetClockInfo(self.h, n.NVML_CLOCK_SM)))
        try:
            bits = n.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except AttributeError:
            bits = n.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        for name, bit in self.NVML_BITS.items():
            if bits & bit:
                self.reasons.add(name)

    def _poll_nvml(self):
        while not self.stop.wait(0.002):
            try:
                self._sample_nvml()
            except Exception:
                return

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.nvml is not None:
            self._sample_nvml()  # and one at the end
            self.stop.set()
            self.t.join(timeout=1)
            return
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.nvml is not None:
            return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                    "sm_max_mhz": max(self.mx) if self.mx else None, "reasons": sorted(self.reasons),
                    "samples": len(self.sm), "source": "nvml (2 ms polling during the timed region)"}
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) >= 8:
                for n, v in zip(names, r[4:8]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi -lms 100"}


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _bf16(t_bits, torch, device):
    return torch.from_numpy(np.ascontiguousarray(t_bits).view(np.int16)).view(torch.bfloat16).to(device)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2602_06932_b200 import aurora as A
    from paper_2602_06932_b200.build import build

    ws, rank, local = _dist_env()
    if ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    if rank == 0:
        build()
    if ws > 1:
        dist.barrier()
    A.lib()

    cfg = tracegen.CONFIGS[args.config]
    # Multi-GPU (N > 1), weak scaling (per-GPU GEMM work = the 1-GPU config's M x V):
    #   VP (default, the north star's box-level scheme): one global batch of N x R requests,
    #     rank p holds vocab slice p of W and T; only per-row scalars (C1, C3) and the dH
    #     partials (C4) cross NVLink;
    #   DP (--parallel dp): each rank its own batch over the full vocabulary (C2 counts, C5
    #     dW allreduce);
    #   --vp A --dp B (A x B = N): the 2-D layout (the tree config's DP2 x VP4): B DP groups
    #     of A x R requests, each split over A vocab slices.
    if ws > 1:
        if args.vp or args.dp:
            n_vp, n_dp = (args.vp or ws // max(args.dp, 1)), (args.dp or ws // max(args.vp, 1))
        else:
            n_vp, n_dp = (ws, 1) if args.parallel == "vp" else (1, ws)
        if n_vp * n_dp != ws:
            raise SystemExit(f"--vp {n_vp} x --dp {n_dp} != WORLD_SIZE {ws}")
    else:
        n_vp, n_dp = 1, 1
    vp_rank, dp_rank = rank % n_vp, rank // n_vp
    vp = n_vp > 1
    cfg_g = dataclasses.replace(cfg, R=cfg.R * n_vp)   # this DP group's requests
    R, N, d, V, M = cfg_g.R, cfg_g.N, cfg_g.d, cfg_g.V, cfg_g.M
    v0, v1 = vp_rank * V // n_vp, (vp_rank + 1) * V // n_vp
    V_local = v1 - v0
    sparse = bool(args.target_topk)
    if ws == 1:
        tr = (tracegen.gen_trace_topk(cfg, K_t=args.target_topk) if sparse else tracegen.gen_trace(cfg))
        W = _bf16(tr["W_bits"], torch, dev)
        T = None if sparse else _bf16(tr["T_bits"], torch, dev)
    else:
        if sparse:
            raise SystemExit("--target-topk is a single-GPU workload")
        # the group's tokens / tree / H from tracegen (seed per DP group, shared by its VP
        # ranks); this rank's W and T slices drawn on the device (same distributions: W ~
        # N(0, (2/sqrt d)^2), T ~ N(0, 2^2) with the designated token planted as the strict
        # row maximum) -- the full [M, V] T of a global batch does not fit host RAM at 8 GPUs
        tr = tracegen.gen_trace(cfg_g, seed=cfg.seed + 1000 * dp_rank, gen_T=False, gen_W=False)
        g = torch.Generator(device=dev).manual_seed(cfg.seed * 1000003 + 7919 * dp_rank + vp_rank)
        W = (torch.randn(V_local, d, generator=g, device=dev) * (2.0 / math.sqrt(d))).to(torch.bfloat16)
        T = torch.empty(M, V_local, dtype=torch.bfloat16, device=dev)
        for m0 in range(0, M, 2048):
            m1 = min(M, m0 + 2048)
            T[m0:m1] = (torch.randn(m1 - m0, V_local, generator=g, device=dev) * 2.0).to(torch.bfloat16)
        des = torch.from_numpy(tr["designated"].astype(np.int64)).to(dev)
        own = torch.nonzero((des >= v0) & (des < v1)).flatten()
        T[own, des[own] - v0] = 16.0           # > every N(0, 4) draw of the row: strict maximum
        del des, own

    comm = None
    if ws > 1:
        uid = A.aurora_comm_get_unique_id() if rank == 0 else bytes(128)
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        comm = A.aurora_comm_create(obj[0], ws, rank, n_vp, n_dp)
    elif args.comm1:  # 1-rank communicator: every exchange runs (as an identity) on one GPU
        comm = A.aurora_comm_create(A.aurora_comm_get_unique_id(), 1, 0, 1, 1)

    if sparse:
        Tk_idx = torch.from_numpy(tr["Tk_idx"]).to(dev)
        Tk_val = _bf16(tr["Tk_bits"], torch, dev)
    H = _bf16(tr["H_bits"], torch, dev)
    draft = torch.from_numpy(tr["draft_tokens"]).to(dev)
    parents = None if tr["parents"] is None else torch.from_numpy(tr["parents"]).to(dev)
    num_nodes = None if tr["num_nodes"] is None else torch.from_numpy(tr["num_nodes"]).to(dev)
    st = A.SpecTrainStep(R, N, d, V, V_local=V_local, vocab_offset=v0, comm=comm, device=dev,
                         k_accept=args.k_accept, k_discard=args.k_discard, accept_loss=args.accept_loss,
                         ntp_beta=args.ntp_beta, discard_loss=args.discard_loss)
    if sparse and A.aurora_workspace_size(A.OP_VERIFY, M, d, args.target_topk, st.cfg) > st.ws_bytes:
        raise SystemExit("workspace too small for --target-topk")
    dH = torch.empty(M, d, dtype=torch.float32, device=dev)
    dW = torch.empty(V_local, d, dtype=torch.float32, device=dev)
    opt = None
    sharded = n_dp > 1 and args.optimizer is not None
    if args.optimizer == "fused" and n_dp > 1:
        raise SystemExit("--optimizer fused needs a DP group of 1 (DP: the sharded optimizer, --optimizer)")
    if sharded:  # F3 DP half: reduce-scatter of dW + the optimizer state sharded over the DP group
        opt = A.ShardedAdamW(W.float().reshape(-1), comm, dp_rank, n_dp, lr=1e-5, warmup_steps=400)
    elif args.optimizer:  # F3: fp32 master lm_head + AdamW; the GEMMs read its bf16 copy
        opt = A.AdamW(W.float().reshape(-1), lr=1e-5, warmup_steps=400, comm=comm)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        if opt is not None and args.optimizer == "fused":
            if sparse:
                st.verify_topk(draft, Tk_idx, Tk_val, parents, num_nodes)
            else:
                st.verify(draft, T, parents, num_nodes)
            st.forward(H, W)
            st.backward_adamw(H, W, dH, opt)
            return
        if sparse:
            st.verify_topk(draft, Tk_idx, Tk_val, parents, num_nodes)
        else:
            st.verify(draft, T, parents, num_nodes)
        st.forward(H, W)
        st.backward(H, W, dH, dW, dp_reduce=not sharded)
        if sharded:
            opt.step(dW.reshape(-1), W.reshape(-1))
        elif opt is not None and args.optimizer == "unfused":
            opt.step(dW.reshape(-1), W_bf16=W.reshape(-1))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    assert int(st.status.item()) == 0, "device status word set"

    # ---------------- timed region (device-resident inputs)
    # Default: one step is captured once into a CUDA graph (the C-ABI is stream-ordered with
    # no host syncs) and each of the K timed steps is one replay, bracketed by its CUDA events
    # after the L2 flush -- launch gaps leave the step.  The library's per-phase events are
    # captured as external event nodes, re-timed by every replay and read after each one
    # (aurora_profile_peek), so phase times stay live inside the timed region.  --eager:
    # the steps are launched directly.
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launch_mode = "eager"
    graph = None
    launches_per_step = None
    # multi-rank steps are captured too: the library's collectives are NCCL calls on the
    # caller's stream, which NCCL supports inside CUDA-graph capture (eager on failure)
    if not args.eager:
        try:
            A.aurora_profile_read()  # clear
            A.aurora_profile_enable(True)
            n0 = A.aurora_launch_count()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                step()
            launches_per_step = A.aurora_launch_count() - n0
            A.aurora_profile_enable(False)
            graph.replay()  # untimed: graph upload
            torch.cuda.synchronize()
            launch_mode = "cuda_graph (one step captured once; each timed step is one replay)"
        except Exception as e:  # capture failure falls back to eager
            A.aurora_profile_enable(False)
            A.aurora_profile_read()
            graph = None
            launch_mode = f"eager (graph capture failed: {type(e).__name__})"
    if graph is None:
        A.aurora_profile_read()  # clear
        A.aurora_profile_enable(True)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = A.aurora_launch_count()
    phase_acc = {}
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            evs[i][0].record(stream)
            if graph is not None:
                graph.replay()
            else:
                step()
            evs[i][1].record(stream)
            if graph is not None:  # this replay's phase times (the sync sits outside the events)
                torch.cuda.synchronize()
                for k, (t, n) in A.aurora_profile_read(peek=True).items():
                    a = phase_acc.setdefault(k, [0.0, 0])
                    a[0] += t
                    a[1] += n
        torch.cuda.synchronize()
    if graph is None:
        n_launch = A.aurora_launch_count() - n0
        A.aurora_profile_enable(False)
        phases = A.aurora_profile_read()
    else:
        n_launch = launches_per_step * args.steps
        phases = {k: (v[0], v[1]) for k, v in phase_acc.items()}
        A.aurora_profile_read()  # release the captured events
    ms = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    tokens_per_s = M * n_dp / (ms_step / 1e3)   # n_dp groups of M rows (each split over n_vp vocab slices)

    # ---------------- e2e: public API with pinned host inputs, result read back
    if ws > 1 and not sparse:   # the e2e leg streams this rank's T slice from pinned host memory
        tr = dict(tr, T_bits=T.view(torch.int16).cpu().numpy().view(np.uint16))
    e2e = None if opt is not None else _run_e2e(args, torch, dist, st, tr, W, dH, dW, dev, ws, flush, sparse,
                                                 rows_total=M * n_dp)

    if rank != 0:
        if comm is not None:
            A.aurora_comm_destroy(comm)
        if ws > 1:
            dist.destroy_process_group()
        return

    peak_burst, peak_sus, hbm, peak_src = _peaks()
    # traffic: only for the exact workload the committed ncu capture ran (default objective)
    plain = (not sparse and args.k_accept == 1 and args.k_discard == 10 and args.accept_loss == "fkl"
             and args.optimizer != "fused" and args.discard_loss == "full")
    cfg_dev = dataclasses.replace(cfg_g, V=V_local)  # the work one GPU does (its rows x its vocab slice)
    roof = _roofline(phases, cfg_dev, args.steps, peak_burst, peak_src, hbm,
                     workload=cfg.name if (plain and not vp and ws == 1) else None, optimizer=args.optimizer)
    out = {
        "metric": "speculator-training tokens/s (verify + lm_head fwd/bwd + Eq.3 loss), % bf16 tensor peak",
        "value": round(tokens_per_s, 1),
        "unit": "tokens/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (tracegen seeded traces; random-init lm_head)",
        "config": {"workload": cfg.name + (f"+topk{args.target_topk}" if sparse else ""), "R": R, "N": N,
                   "M_rows_per_dp_group": M, "M_rows_total": M * n_dp, "d": d, "V": V,
                   "target": f"top-{args.target_topk} (id, logit) pairs per row (F1)" if sparse else "dense bf16 logits",
                   "k_accept": args.k_accept, "k_discard": args.k_discard, "accept_loss": args.accept_loss,
                   "ntp_beta": args.ntp_beta, "discard_loss": args.discard_loss,
                   "optimizer": f"adamw ({args.optimizer}, F3)" if args.optimizer else None,
                   "tree": cfg.tree,
                   "parallelism": (f"dp{n_dp}xvp{n_vp} ({n_dp} DP group(s) of {R} requests, lm_head vocab-"
                                   f"parallel over {n_vp})" + (", sharded AdamW" if sharded else "") if ws > 1 else
                                   ("single (1-rank comm)" if args.comm1 else "single")),
                   "inputs": ("tracegen (seeded host draw)" if ws == 1 else
                              "tracegen tokens/tree/H per DP group; W and T slices drawn on the device (seeded "
                              "N(0,(2/sqrt d)^2) / N(0,4) with the designated token planted at 16.0)"),
                   "V_local": V_local,
                   "l2": "flushed between timed steps (256 MiB write outside the step events)",
                   "launch": launch_mode},
        "gpu_launches": int(n_launch),
        "phases_ms_per_step": {k: round(v[0] / args.steps, 4) for k, v in phases.items() if v[1]},
        "roofline": roof,
        "e2e": e2e,
        "clocks": clk.summary(),
    }
    # executed GEMM flops over the step against the BURST bf16 peak (MEASURED_PEAKS.json
    # bf16_tflops; the sustained figure is the power-capped 4 s loop): 6MVd (fwd, dW, dH) on
    # the staged path, 8MVd when the backward recomputes Z (dz GEMM)
    gemms = 4 if "bwd_dz_gemm" in phases and phases["bwd_dz_gemm"][1] else 3
    flops_step = 2.0 * gemms * M * V_local * d
    out["executed_gemm_flops_per_step"] = flops_step
    out["tensor_frac_step"] = round((flops_step / (ms_step / 1e3)) / (peak_burst * 1e12), 4)
    out["tensor_frac_step_vs_sustained"] = round((flops_step / (ms_step / 1e3)) / (peak_sus * 1e12), 4)
    out["algorithmic_tensor_frac_step"] = round((6.0 * M * V_local * d / (ms_step / 1e3)) / (peak_burst * 1e12), 4)
    if not args.no_cpu_baseline:
        out["cpu_baseline"] = _cpu_baseline(cfg, args)
    print(json.dumps(out), flush=True)
    if comm is not None:
        A.aurora_comm_destroy(comm)
    if ws > 1:
        dist.destroy_process_group()


def _run_e2e(args, torch, dist, st, tr, W, dH, dW, dev, ws, flush, sparse=False, rows_total=None):
    """Same step through the public API (SpecTrainStep), with the trace batch (T -- or,
    sparse, the top-K (id, logit) payload the paper transmits, P:391-392 --, H, draft
    tokens, parents, ragged counts) copied H2D from pinned host memory every step and the
    step's result (loss, accept lengths) read back D2H.  The copy of step i+1 runs on a
    second stream into the other half of a double buffer while step i computes -- all of
    it inside the timed region."""
    keys = ("Tk_idx", "Tk_bits") if sparse else ("T_bits",)
    hostb = {k: torch.from_numpy(np.ascontiguousarray(tr[k]).view(np.int16 if k.endswith("bits") else np.int32))
             .pin_memory() for k in keys + ("H_bits", "draft_tokens", "parents", "num_nodes")
             if tr[k] is not None}
    bufs = [{k: torch.empty(v.shape, dtype=v.dtype, device=dev) for k, v in hostb.items()} for _ in range(2)]
    outs = [(torch.empty(1, dtype=torch.float32).pin_memory(), torch.empty(st.R, dtype=torch.int32).pin_memory())
            for _ in range(2)]
    h2d = sum(v.numel() * v.element_size() for v in hostb.values())
    d2h = 4 + st.R * 4
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]

    def as_bf16(t):
        return t.view(torch.bfloat16)

    def run(n):
        for i in range(n):
            b = i & 1
            with torch.cuda.stream(copy):
                if i >= 2:
                    copy.wait_event(consumed[b])
                for k, v in hostb.items():
                    bufs[b][k].copy_(v, non_blocking=True)
                copied[b].record(copy)
            comp.wait_event(copied[b])
            B = bufs[b]
            if sparse:
                st.verify_topk(B["draft_tokens"], B["Tk_idx"], as_bf16(B["Tk_bits"]), B.get("parents"),
                               B.get("num_nodes"))
                st.forward(as_bf16(B["H_bits"]), W)
                st.backward(as_bf16(B["H_bits"]), W, dH, dW)
            else:
                st.step(B["draft_tokens"], as_bf16(B["T_bits"]), as_bf16(B["H_bits"]), W, dH, dW,
                        B.get("parents"), B.get("num_nodes"))
            consumed[b].record(comp)
            outs[b][0].copy_(st.loss, non_blocking=True)
            outs[b][1].copy_(st.accept_len, non_blocking=True)

    run(max(3, args.warmup))
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(comp)
    copy.wait_event(e0)
    run(args.steps)
    comp.wait_stream(copy)
    e1.record(comp)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    rows_total = st.M * ws if rows_total is None else rows_total
    return {"value": round(rows_total / (ms_step / 1e3), 1), "unit": "tokens/s", "ms_per_step": round(ms_step, 4),
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "note": "pinned H2D of step i+1 overlapped with step i on a copy stream (double buffer); "
                    "no L2 flush (each step streams its trace from host)"}


def _phase_work(cfg, k, launches_per_step):
    """Algorithmic work of one launch of GEMM phase k (SURVEY 8(d) per-unit figures):
    flops = 2 d per (row, vocab column); bytes = the phase's compulsory DRAM traffic."""
    M, V, d = cfg.M, cfg.V, cfg.d
    vc = V / launches_per_step               # vocab columns per launch (chunked phases)
    flops = 2.0 * M * vc * d
    if k == "fwd_gemm":                      # W once, H, (m, s, u) partials
        byts = 2.0 * V * d + 2.0 * M * d + 12.0 * M * 2 * (V / 256.0)
    elif k == "bwd_dz_gemm":                 # W chunk once, H, bf16 dZ^T chunk write
        byts = 2.0 * vc * d + 2.0 * M * d + 2.0 * vc * M
    elif k == "bwd_dw_gemm":                 # fp32 dW chunk write, dZ^T chunk + H reads
        byts = 4.0 * vc * d + 2.0 * vc * M + 2.0 * M * d
    else:                                    # dH: W chunk + dZ^T chunk reads, fp32 dH write
        byts = 2.0 * vc * d + 2.0 * vc * M + 4.0 * M * d
    return flops, byts


def _roofline(phases, cfg, steps, peak, peak_src, hbm_peak_gbs=6551.0, workload=None, optimizer=None):
    """Dominant lm_head kernel (largest share of the step): achieved algorithmic work per
    launch / mean launch time, against whichever roofline bounds it (tensor or HBM)."""
    per = []
    best = None
    for k in ("fwd_gemm", "bwd_dz_gemm", "bwd_dw_gemm", "bwd_dh_gemm", "bwd_fused", "adamw"):
        if k not in phases or phases[k][1] == 0:
            continue
        tot_ms, n = phases[k]
        lps = n / steps
        t = (tot_ms / n) / 1e3
        if k == "adamw" and optimizer == "fused":  # F3 in the dW epilogue: m, v, W read + written, bf16 W
            flops, byts = 2 * 2.0 * cfg.M * cfg.V * cfg.d, 26.0 * cfg.V * cfg.d
        elif k == "adamw":  # F3 unfused: norm pass 4 B + update 30 B per lm_head element
            flops, byts = 0.0, 34.0 * cfg.V * cfg.d
        elif k == "bwd_fused":
            flops, byts = 3 * 2.0 * cfg.M * cfg.V * cfg.d, 4.0 * cfg.V * cfg.d + 4.0 * cfg.V * cfg.d
        else:
            flops, byts = _phase_work(cfg, k, lps)
        t_tensor, t_hbm = flops / (peak * 1e12), byts / (hbm_peak_gbs * 1e9)
        bound = "tensor" if t_tensor >= t_hbm else "hbm"
        rec = {"kernel": k, "ms_per_step": round(tot_ms / steps, 4), "launches_per_step": lps,
               "achieved_tflops": round(flops / t / 1e12, 1), "achieved_gbs": round(byts / t / 1e9, 1),
               "bound": bound, "frac": round(max(t_tensor, t_hbm) / t, 4)}
        per.append(rec)
        if best is None or tot_ms > best[1]:
            best = (k, tot_ms, rec)
    # G2 (target scan) and G6 (row combine) as achieved DRAM GB/s vs the HBM peak
    for k, byts in (("target_scan", 2.0 * cfg.M * cfg.V),
                    ("fwd_combine", 16.0 * cfg.M * 2 * math.ceil(cfg.V / 256.0)),
                    ("bwd_dz_rescale", 4.0 * cfg.M * cfg.V)):
        if k in phases and phases[k][1]:
            tot_ms, n = phases[k]
            t = (tot_ms / steps) / 1e3
            per.append({"kernel": k, "ms_per_step": round(tot_ms / steps, 4), "achieved_gbs": round(byts / t / 1e9, 1),
                        "bound": "hbm", "frac": round(byts / t / 1e9 / hbm_peak_gbs, 4),
                        "work": {"target_scan": "M*V*2 B of T read once",
                                 "fwd_combine": "(m, s, u, r) partials, >= 16 B per (row, 128-column tile half)",
                                 "bwd_dz_rescale": "M*V bf16 staged numerators read + dz written (4 B per element)"}[k]})
    if best is None:
        return None
    k, _, rec = best
    if rec["bound"] == "tensor":
        out = {"bound": "tensor", "kernel": k, "achieved": rec["achieved_tflops"], "peak": peak, "unit": "TFLOP/s",
               "peak_source": f"{peak_src} bf16_tflops (burst, torch.matmul 8192^3 best of 10)",
               "work_per_launch": "2*M*V_chunk*d flops (2 d per row per vocab column, SURVEY 8(d))"}
    else:
        out = {"bound": "hbm", "kernel": k, "achieved": rec["achieved_gbs"], "peak": hbm_peak_gbs, "unit": "GB/s",
               "peak_source": f"{peak_src} hbm_gbs (copy)",
               "work_per_launch": "compulsory DRAM bytes per launch (fp32 dW chunk write + dZ^T/H reads, DESIGN.md 6)"}
    if k == "adamw":
        out["work_per_launch"] = ("26 B per lm_head element (F3 fused: m/v/W fp32 read + write, W bf16 write; dW never "
                                  "stored)" if optimizer == "fused" else
                                  "34 B per lm_head element (F3: dW norm pass + dW/m/v/W reads, m/v/W fp32 + W bf16 writes)")
    out["frac"] = round(out["achieved"] / out["peak"], 4)
    out["traffic"] = _traffic_for(k, workload)
    out["phases"] = per
    return out


def _traffic_for(kernel, workload):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of this kernel from the
    committed ncu --set full capture of this workload (profiles/traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        try:
            v = json.load(open(p)).get(workload, {}).get(kernel)
            return int(v) if v is not None else None
        except Exception:
            return None
    return None


def _cpu_baseline(cfg, args, reqs=None):
    """The oracle as it stands, on a bounded sample (first `reqs` requests of the
    same workload, full vocabulary and hidden size), on this host's cores."""
    import oracle
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"] or [1])
    except Exception:
        cores = len(os.sched_getaffinity(0))
    reqs = reqs or args.cpu_reqs
    tr = tracegen.gen_trace(cfg)
    sub = _subsample(tr, reqs)
    t0 = time.perf_counter()
    oracle.step(sub)
    dt = time.perf_counter() - t0
    return {"value": round(sub["M"] / dt, 2), "unit": "tokens/s", "cores": int(cores), "kind": "oracle",
            "sample": f"first {reqs} of {cfg.R} requests ({sub['M']} rows) of '{cfg.name}', full V={cfg.V}, "
                      f"d={cfg.d}; verify+fwd+bwd f64; {dt:.2f} s"}


def _subsample(tr, reqs):
    cfg = tr["cfg"]
    rows = reqs * (cfg.N + 1)
    sub = dict(tr)
    sub["draft_tokens"] = tr["draft_tokens"][:reqs]
    sub["parents"] = None if tr["parents"] is None else tr["parents"][:reqs]
    sub["num_nodes"] = None if tr["num_nodes"] is None else tr["num_nodes"][:reqs]
    sub["T_bits"] = tr["T_bits"][:rows]
    sub["H_bits"] = tr["H_bits"][:rows]
    sub["M"] = rows
    sub["R"] = reqs
    return sub


def run_reference(args):
    ws, rank, _ = _dist_env()
    if rank != 0:
        return
    cfg = tracegen.CONFIGS[args.config]
    tr = tracegen.gen_trace(cfg)
    sub = _subsample(tr, args.ref_reqs)
    import oracle
    for _ in range(args.warmup if args.warmup_ref else 0):
        oracle.step(sub)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.step(sub)
    dt = (time.perf_counter() - t0) / args.steps
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"] or [1])
    except Exception:
        cores = len(os.sched_getaffinity(0))
    val = round(sub["M"] / dt, 2)
    out = {"impl": "reference", "metric": "speculator-training tokens/s (verify + lm_head fwd/bwd + Eq.3 loss), "
           "% bf16 tensor peak", "value": val, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (tracegen seeded traces)",
           "config": {"workload": cfg.name, "R": cfg.R, "N": cfg.N, "d": cfg.d, "V": cfg.V,
                      "parallelism": "cpu oracle (rank 0 only)"},
           "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": int(cores), "kind": "oracle",
                            "sample": f"first {args.ref_reqs} of {cfg.R} requests ({sub['M']} rows) per step, "
                                      f"full V and d"},
           "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------------------- NEXT F4
def _ta_work(meta):
    """Algorithmic work of one tree-attention fwd+bwd over a batch (F4):
    visible (row, key) pairs per query head -- every prefix key for each valid tree row plus
    the row's ancestor closure -- times 4 dh flops forward and 10 dh backward (S, dP, dV, dQ,
    dK); compulsory DRAM bytes: Q, K/V (prefix + tree) read once per kernel that needs them,
    O/lse written, dO/O/lse read, dQ fp32 and dK/dV bf16 written."""
    c = meta["cfg"]
    off = meta["prefix_off"]
    lens = np.diff(off).astype(np.int64)
    N1 = c.N + 1
    pairs = 0
    for r in range(c.R):
        nn = c.N if meta["num_nodes"] is None else int(meta["num_nodes"][r])
        par = None if meta["parents"] is None else meta["parents"][r]
        depth_sum = 1                                   # root sees itself
        for n in range(nn):
            d, p = 2, (n - 1 if par is None else int(par[n]))
            while p >= 0:
                d += 1
                p = p - 1 if par is None else int(par[p])
            depth_sum += d
        pairs += (nn + 1) * int(lens[r]) + depth_sum
    pairs *= c.Hq
    rows = c.R * N1
    q_b = rows * c.Hq * c.dh * 2
    kv_b = (int(lens.sum()) + rows) * c.Hkv * c.dh * 2 * 2       # K and V
    fwd_b = q_b + kv_b + q_b + rows * c.Hq * 4                    # + O + lse
    dq_b = 3 * q_b + rows * c.Hq * 8 + kv_b + 2 * q_b             # Q, dO, O(dsum), lse+Dsum, K/V, dQ fp32
    dkdv_b = kv_b + kv_b + 2 * q_b + rows * c.Hq * 8              # K/V read, dK/dV write, Q/dO, lse/Dsum
    fused_b = 3 * q_b + rows * c.Hq * 8 + kv_b + 2 * q_b + kv_b   # Q, dO, O, lse+Dsum, K/V, dQ, dK/dV
    return dict(pairs=pairs, fwd_flops=4.0 * c.dh * pairs, bwd_flops=10.0 * c.dh * pairs, fwd_bytes=fwd_b,
                dq_bytes=dq_b, dkdv_bytes=dkdv_b, fused_bytes=fused_b, rows=rows)


def run_tree_attn(args):
    """F4 bench: tree-attention fwd + bwd of the draft layer over a batch of speculative trees
    with ragged cached prefixes (tracegen TREE_ATTN_CONFIGS; values drawn on the device from a
    seeded generator with the distributions of tracegen.gen_tree_attn)."""
    import torch
    from paper_2602_06932_b200 import aurora as A
    from paper_2602_06932_b200.build import build

    import torch.distributed as dist
    # N > 1: requests are independent (no exchange step exists), so every rank attends its own
    # batch of trees (weak scaling, its own seed) and no collective touches the data path; the
    # barrier + max-over-ranks timing follows the bench contract.
    ws, rank, local = _dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    if rank == 0:
        build()
    if ws > 1:
        dist.barrier()
    A.lib()
    meta = tracegen.gen_tree_attn_meta(args.ta_config)
    c = meta["cfg"]
    N1 = c.N + 1
    off = meta["prefix_off"]
    P = int(off[-1])
    g = torch.Generator(device=dev)
    g.manual_seed(c.seed + 7919 * rank)
    qscale = torch.ones(c.Hq, 1, device=dev)
    G = c.Hq // c.Hkv
    for h in range(c.Hq):
        if (h // G) % 4 == 3:
            qscale[h] = 3.0

    def rnd(*shape, scale=1.0):
        return (torch.randn(*shape, generator=g, device=dev, dtype=torch.float32) * scale).to(torch.bfloat16)

    Q = (torch.randn(c.R, N1, c.Hq, c.dh, generator=g, device=dev) * qscale).to(torch.bfloat16)
    Kt, Vt = rnd(c.R, N1, c.Hkv, c.dh), rnd(c.R, N1, c.Hkv, c.dh)
    Kp, Vp = rnd(P, c.Hkv, c.dh), rnd(P, c.Hkv, c.dh)
    dO = rnd(c.R, N1, c.Hq, c.dh, scale=0.1)
    poff = torch.from_numpy(off.astype(np.int32)).to(dev)
    par = None if meta["parents"] is None else torch.from_numpy(meta["parents"].astype(np.int32)).to(dev)
    nn = None if meta["num_nodes"] is None else torch.from_numpy(meta["num_nodes"].astype(np.int32)).to(dev)
    max_prefix = int(np.diff(off).max())
    ta = A.TreeAttention(c.R, c.N, c.Hq, c.Hkv, c.dh, poff, max_prefix, parents=par, num_nodes=nn)
    O = torch.empty_like(Q)
    lse = torch.empty(c.R, N1, c.Hq, dtype=torch.float32, device=dev)
    dQ = torch.empty(Q.shape, dtype=torch.float32, device=dev)
    dKt, dVt, dKp, dVp = (torch.empty_like(x) for x in (Kt, Vt, Kp, Vp))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(q=Q, kt=Kt, vt=Vt, kp=Kp, vp=Vp, do=dO):
        ta.forward(q, kt, vt, kp, vp, O, lse)
        ta.backward(q, kt, vt, kp, vp, O, lse, do, dQ, dKt, dVt, dKp, dVp)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    assert int(ta.status.item()) == 0
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    A.aurora_profile_read()
    A.aurora_profile_enable(True)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = A.aurora_launch_count()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    n_launch = A.aurora_launch_count() - n0
    A.aurora_profile_enable(False)
    phases = A.aurora_profile_read()
    t_ms = torch.tensor([sum(a.elapsed_time(b) for a, b in evs)], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
        dist.barrier()
    ms_step = float(t_ms.item()) / args.steps
    w = _ta_work(meta)
    rows_per_s = w["rows"] * ws / (ms_step / 1e3)   # every rank's batch counts

    # e2e: every step copies its inputs from pinned host memory and reads lse back
    host = {k: v.cpu().pin_memory() for k, v in dict(Q=Q, Kt=Kt, Vt=Vt, Kp=Kp, Vp=Vp, dO=dO).items()}
    lse_h = torch.empty(lse.shape, dtype=torch.float32).pin_memory()
    h2d = sum(v.numel() * v.element_size() for v in host.values())
    e_steps = max(2, min(args.steps, 5))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e_steps):
        dv = {k: v.to(dev, non_blocking=True) for k, v in host.items()}
        step(dv["Q"], dv["Kt"], dv["Vt"], dv["Kp"], dv["Vp"], dv["dO"])
        lse_h.copy_(lse, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e_ms = torch.tensor([e0.elapsed_time(e1) / e_steps], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e_ms.item())
    if rank != 0:
        dist.destroy_process_group()
        return

    _, _, hbm, peak_src = _peaks()
    per = []
    for k, byts, flops in (("tree_attn_fwd", w["fwd_bytes"], w["fwd_flops"]),
                           ("tree_attn_fwd_tc", w["fwd_bytes"], w["fwd_flops"]),
                           ("tree_attn_bwd_dq", w["dq_bytes"], 0.4 * w["bwd_flops"]),
                           ("tree_attn_bwd_dkdv", w["dkdv_bytes"], 0.6 * w["bwd_flops"]),
                           ("tree_attn_bwd_fused", w["fused_bytes"], w["bwd_flops"])):
        if k in phases and phases[k][1]:
            t = phases[k][0] / args.steps / 1e3
            per.append({"kernel": k, "ms_per_step": round(t * 1e3, 4), "achieved_gbs": round(byts / t / 1e9, 1),
                        "achieved_tflops": round(flops / t / 1e12, 1), "frac_hbm": round(byts / t / 1e9 / hbm, 4)})
    dom = max(per, key=lambda x: x["ms_per_step"])
    out = {
        "metric": "tree-attention fwd+bwd tokens/s (F4 draft-layer attention, ancestor-closure mask)",
        "value": round(rows_per_s, 1), "unit": "tokens/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (seeded device generator; tracegen structure)",
        "config": {"workload": c.name, "R": c.R, "N": c.N, "Hq": c.Hq, "Hkv": c.Hkv, "dh": c.dh,
                   "prefix_tokens": P, "max_prefix": max_prefix, "tree": c.tree,
                   "visible_pairs_per_head_avg": round(w["pairs"] / c.Hq / c.R, 1),
                   "l2": "flushed between timed steps (256 MiB write outside the step events)", "launch": "eager",
                   "parallelism": f"dp{ws} (independent tree batches per rank, no collective)" if ws > 1 else "single"},
        "gpu_launches": int(n_launch),
        "phases_ms_per_step": {k: round(v[0] / args.steps, 4) for k, v in phases.items() if v[1]},
        "roofline": {"bound": "hbm", "kernel": dom["kernel"], "achieved": dom["achieved_gbs"], "peak": hbm,
                     "unit": "GB/s", "frac": round(dom["achieved_gbs"] / hbm, 4),
                     "traffic": _traffic_for(dom["kernel"], c.name),
                     "peak_source": f"{peak_src} hbm_gbs (copy)",
                     "work_per_launch": "compulsory DRAM bytes (prefix+tree K/V, Q/dO/O, outputs), DESIGN.md §6 F4",
                     "phases": per},
        "e2e": {"value": round(w["rows"] * ws / (e2e_ms / 1e3), 1), "unit": "tokens/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(lse.numel() * 4)},
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline and ws == 1:
        from oracle import tree_attention as TA
        reqs = list(range(min(4, c.R)))
        sub = tracegen.gen_tree_attn(c.name, requests=reqs)
        t0 = time.perf_counter()
        TA.fwd_bwd(sub)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": round(len(reqs) * N1 / dt, 2), "unit": "tokens/s",
                               "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
                               "sample": f"first {len(reqs)} of {c.R} requests of '{c.name}', fwd+bwd f64; {dt:.2f} s"}
    print(json.dumps(out), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def run_draft_layer(args):
    """F4 bench: the whole EAGLE-3 draft layer (fc + decoder layer with tree RoPE and tree
    attention), fwd + bwd, over the F4 tree workloads with the target's dense shapes (d = 4096;
    MLP 14336 for the Llama-3.1-8B speculator, 12288 for Qwen3-8B).  Weights/inputs drawn on the
    device from a seeded generator (N(0, 1/fan_in) weights, N(0, 1) inputs)."""
    import torch
    from paper_2602_06932_b200 import aurora as A
    from paper_2602_06932_b200.build import build

    ws, rank, local = _dist_env()
    if rank != 0:        # measured on one GPU (requests are independent; see run_tree_attn for N > 1)
        return
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    build()
    A.lib()
    meta = tracegen.gen_tree_attn_meta(args.ta_config)
    c = meta["cfg"]
    d, I = 4096, (14336 if c.name == "ta_llama" else 12288)
    N1 = c.N + 1
    M = c.R * N1
    off = meta["prefix_off"]
    P = int(off[-1])
    g = torch.Generator(device=dev)
    g.manual_seed(c.seed + 17)
    rnd = lambda *s, k=1.0: (torch.randn(*s, generator=g, device=dev) * k).to(torch.bfloat16)
    qd, kd = c.Hq * c.dh, c.Hkv * c.dh
    W = dict(Wfc=rnd(d, 3 * d, k=(3 * d) ** -0.5), Wq=rnd(qd, 2 * d, k=(2 * d) ** -0.5),
             Wk=rnd(kd, 2 * d, k=(2 * d) ** -0.5), Wv=rnd(kd, 2 * d, k=(2 * d) ** -0.5), Wo=rnd(d, qd, k=qd ** -0.5),
             Wg=rnd(I, d, k=d ** -0.5), Wu=rnd(I, d, k=d ** -0.5), Wd=rnd(d, I, k=I ** -0.5),
             we=torch.ones(d, device=dev), wh=torch.ones(d, device=dev), wpost=torch.ones(d, device=dev),
             wfinal=torch.ones(d, device=dev))
    h3, e = rnd(M, 3 * d), rnd(M, d)
    Kp, Vp = rnd(P, c.Hkv, c.dh), rnd(P, c.Hkv, c.dh)
    dH = torch.randn(M, d, generator=g, device=dev) * 0.1
    poff = torch.from_numpy(off.astype(np.int32)).to(dev)
    par = None if meta["parents"] is None else torch.from_numpy(meta["parents"].astype(np.int32)).to(dev)
    nn = None if meta["num_nodes"] is None else torch.from_numpy(meta["num_nodes"].astype(np.int32)).to(dev)
    ta = A.TreeAttention(c.R, c.N, c.Hq, c.Hkv, c.dh, poff, int(np.diff(off).max()), parents=par, num_nodes=nn)
    layer = A.DraftLayer(ta, d, I, W, theta=500000.0 if c.name == "ta_llama" else 1000000.0, eps=1e-6)
    H = torch.empty(M, d, dtype=torch.bfloat16, device=dev)
    G = {k: torch.empty(v.shape, dtype=torch.float32, device=dev) for k, v in W.items()}
    dh3 = torch.empty(M, 3 * d, dtype=torch.float32, device=dev)
    de = torch.empty(M, d, dtype=torch.float32, device=dev)
    dKp, dVp = torch.empty_like(Kp), torch.empty_like(Vp)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        layer.forward(h3, e, Kp, Vp, H)
        layer.backward(h3, e, Kp, Vp, dH, G, dh3, de, dKp, dVp)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    assert int(ta.status.item()) == 0
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    # one step captured into a CUDA graph (the layer is stream-ordered: cuBLAS + library kernels,
    # no host syncs); each timed step is one replay, per-phase events re-timed by every replay
    graph, launch_mode = None, "eager"
    if not args.eager:
        try:
            A.aurora_profile_read()
            A.aurora_profile_enable(True)
            n0 = A.aurora_launch_count()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                step()
            per_step = A.aurora_launch_count() - n0
            A.aurora_profile_enable(False)
            graph.replay()
            torch.cuda.synchronize()
            launch_mode = "cuda_graph (one step captured once; each timed step is one replay)"
        except Exception as ex:
            A.aurora_profile_enable(False)
            A.aurora_profile_read()
            graph, launch_mode = None, f"eager (graph capture failed: {type(ex).__name__})"
    if graph is None:
        A.aurora_profile_read()
        A.aurora_profile_enable(True)
    n0 = A.aurora_launch_count()
    acc = {}
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            evs[i][0].record(stream)
            if graph is not None:
                graph.replay()
            else:
                step()
            evs[i][1].record(stream)
            if graph is not None:
                torch.cuda.synchronize()
                for k, (t, n) in A.aurora_profile_read(peek=True).items():
                    a_ = acc.setdefault(k, [0.0, 0])
                    a_[0] += t
                    a_[1] += n
        torch.cuda.synchronize()
    if graph is None:
        n_launch = A.aurora_launch_count() - n0
        A.aurora_profile_enable(False)
        phases = A.aurora_profile_read()
    else:
        n_launch = per_step * args.steps
        phases = {k: (v[0], v[1]) for k, v in acc.items()}
        A.aurora_profile_read()
    ms_step = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    w = _ta_work(meta)
    gemm_fwd = 2.0 * M * (3 * d * d + 2 * d * (qd + 2 * kd) + qd * d + 3 * d * I)
    flops = 3.0 * gemm_fwd + w["fwd_flops"] + w["bwd_flops"]
    peak_burst, peak_sus, hbm, peak_src = _peaks()
    achieved = flops / (ms_step / 1e3) / 1e12
    attn_ms = sum(v[0] for k, v in phases.items() if k.startswith("tree_attn")) / args.steps
    out = {
        "metric": "draft-layer fwd+bwd tokens/s (F4: EAGLE-3 fc + decoder layer with tree RoPE + tree attention)",
        "value": round(M / (ms_step / 1e3), 1), "unit": "tokens/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded device generator; tracegen structure)",
        "config": {"workload": c.name + "+draft_layer", "R": c.R, "N": c.N, "d": d, "I": I, "Hq": c.Hq, "Hkv": c.Hkv,
                   "dh": c.dh, "prefix_tokens": P, "gemm": "libaurora tcgen05 engine (bf16 / fp32 TMA-store epilogues)",
                   "l2": "flushed between timed steps (256 MiB write outside the step events)", "launch": launch_mode},
        "gpu_launches": int(n_launch),
        "phases_ms_per_step": {k: round(v[0] / args.steps, 4) for k, v in phases.items() if v[1]},
        "roofline": {"bound": "tensor", "kernel": "draft_layer_step", "achieved": round(achieved, 1),
                     "peak": peak_burst, "unit": "TFLOP/s", "frac": round(achieved / peak_burst, 4), "traffic": None,
                     "peak_source": f"{peak_src} bf16_tflops (burst)",
                     "frac_vs_sustained": round(achieved / peak_sus, 4),
                     "work_per_launch": "3 x dense GEMM flops of the layer (fwd + 2 bwd) + tree attention 14 dh per pair",
                     "attention_ms_per_step": round(attn_ms, 4)},
        "clocks": clk.summary(),
    }
    print(json.dumps(out), flush=True)


def run_full_step(args):
    """Whole speculator training step on one GPU: greedy verification + labels -> F4 draft layer
    (fc + decoder layer with tree RoPE + tree attention) -> H -> lm_head fwd/bwd with the Eq. 3
    loss -> dH -> draft layer bwd (SpeculatorStep).  Trace (T, draft tokens, tree) from tracegen's
    `--config` workload; cached prefixes from the matching F4 workload (ta_llama for llama, ta_tree
    otherwise); layer weights / inputs from a seeded device generator."""
    import torch
    from paper_2602_06932_b200 import aurora as A
    from paper_2602_06932_b200.build import build

    ws, rank, local = _dist_env()
    if rank != 0:
        return
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    build()
    A.lib()
    cfg = tracegen.CONFIGS[args.config]
    tr = tracegen.gen_trace(cfg)
    R, N, d, V, M = cfg.R, cfg.N, cfg.d, cfg.V, cfg.M
    meta = tracegen.gen_tree_attn_meta("ta_llama" if args.config == "llama" else "ta_tree")
    ca = meta["cfg"]
    off = meta["prefix_off"][:R + 1]
    P = int(off[-1])
    I = 14336 if args.config == "llama" else 12288
    g = torch.Generator(device=dev)
    g.manual_seed(cfg.seed + 23)
    rnd = lambda *s, k=1.0: (torch.randn(*s, generator=g, device=dev) * k).to(torch.bfloat16)
    qd, kd = ca.Hq * ca.dh, ca.Hkv * ca.dh
    # every trainable parameter in flat buffers (SpeculatorParams): --optimizer adds ONE AdamW step
    # over lm_head + draft layer per training step (F3 over the whole speculator)
    sp = A.SpeculatorParams(d, I, ca.Hq, ca.Hkv, ca.dh, V, dev)
    fan = dict(Wfc=3 * d, Wq=2 * d, Wk=2 * d, Wv=2 * d, Wo=qd, Wg=d, Wu=d, Wd=I)
    for k_, f_ in fan.items():
        sp.M[k_].copy_(torch.randn(sp.M[k_].shape, generator=g, device=dev) * f_ ** -0.5)
    for k_ in ("we", "wh", "wpost", "wfinal"):
        sp.M[k_].fill_(1.0)
    sp.M["W_lm"].copy_(_bf16(tr["W_bits"], torch, dev).float())
    sp.bf.copy_(sp.master.to(torch.bfloat16))
    W, W_lm = sp.W, sp.W_lm
    opt = sp.adamw(lr=1e-5, warmup_steps=400) if args.optimizer else None
    h3, e = rnd(M, 3 * d), rnd(M, d)
    Kp, Vp = rnd(P, ca.Hkv, ca.dh), rnd(P, ca.Hkv, ca.dh)
    T = _bf16(tr["T_bits"], torch, dev)
    draft = torch.from_numpy(tr["draft_tokens"]).to(dev)
    par = None if tr["parents"] is None else torch.from_numpy(tr["parents"]).to(dev)
    nn = None if tr["num_nodes"] is None else torch.from_numpy(tr["num_nodes"]).to(dev)
    ta = A.TreeAttention(R, N, ca.Hq, ca.Hkv, ca.dh, torch.from_numpy(off.astype(np.int32)).to(dev),
                         int(np.diff(off).max()), parents=par, num_nodes=nn)
    layer = A.DraftLayer(ta, d, I, W, theta=500000.0 if args.config == "llama" else 1000000.0, eps=1e-6)
    spec = A.SpecTrainStep(R, N, d, V, device=dev)
    st = A.SpeculatorStep(spec, layer)
    H = torch.empty(M, d, dtype=torch.bfloat16, device=dev)
    dH = torch.empty(M, d, dtype=torch.float32, device=dev)
    dW_lm, G = sp.dW_lm, sp.G
    dh3 = torch.empty(M, 3 * d, dtype=torch.float32, device=dev)
    de = torch.empty(M, d, dtype=torch.float32, device=dev)
    dKp, dVp = torch.empty_like(Kp), torch.empty_like(Vp)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        st.step(draft, T, h3, e, Kp, Vp, W_lm, H, dH, dW_lm, G, dh3, de, dKp, dVp, parents=par, num_nodes=nn)
        if opt is not None:
            sp.optimizer_step(opt)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    assert int(spec.status.item()) == 0 and int(ta.status.item()) == 0
    graph, launch_mode = None, "eager"
    per_step = None
    if not args.eager:
        try:
            c0 = A.aurora_launch_count()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                step()
            per_step = A.aurora_launch_count() - c0
            graph.replay()
            torch.cuda.synchronize()
            launch_mode = "cuda_graph (one step captured once; each timed step is one replay)"
        except Exception as ex:
            graph, launch_mode = None, f"eager (graph capture failed: {type(ex).__name__})"
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    n0 = A.aurora_launch_count()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            evs[i][0].record(stream)
            graph.replay() if graph is not None else step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    ms_step = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    w = _ta_work(dict(meta, cfg=dataclasses.replace(ca, R=R), prefix_off=off, parents=tr["parents"],
                      num_nodes=tr["num_nodes"]))
    gemm_fwd = 2.0 * M * (3 * d * d + 2 * d * (qd + 2 * kd) + qd * d + 3 * d * I)
    flops = 3.0 * gemm_fwd + w["fwd_flops"] + w["bwd_flops"] + 8.0 * M * V * d   # + lm_head: 4 GEMMs executed
    peak_burst, peak_sus, _, peak_src = _peaks()
    achieved = flops / (ms_step / 1e3) / 1e12
    out = {
        "metric": "whole speculator training step tokens/s (verify + F4 draft layer + lm_head Eq.3 fwd/bwd)",
        "value": round(M / (ms_step / 1e3), 1), "unit": "tokens/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (tracegen trace + seeded device generator)",
        "config": {"workload": cfg.name + "+draft_layer", "optimizer": "adamw over all params (F3)" if opt else None,
                   "params": int(sp.master.numel()), "R": R, "N": N, "d": d, "V": V, "I": I, "Hq": ca.Hq,
                   "Hkv": ca.Hkv, "prefix_tokens": P, "tree": cfg.tree,
                   "l2": "flushed between timed steps (256 MiB write outside the step events)", "launch": launch_mode},
        "gpu_launches": int(per_step * args.steps if graph is not None else A.aurora_launch_count() - n0),
        "roofline": {"bound": "tensor", "kernel": "speculator_step", "achieved": round(achieved, 1), "peak": peak_burst,
                     "unit": "TFLOP/s", "frac": round(achieved / peak_burst, 4), "traffic": None,
                     "peak_source": f"{peak_src} bf16_tflops (burst)",
                     "frac_vs_sustained": round(achieved / peak_sus, 4),
                     "work_per_launch": "executed GEMM flops: 3 x draft-layer dense fwd + 8 M V d lm_head + tree attention"},
        "clocks": clk.summary(),
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="qwen3", choices=sorted(tracegen.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-reqs", type=int, default=8)
    ap.add_argument("--ref-reqs", type=int, default=2)
    ap.add_argument("--warmup-ref", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--target-topk", type=int, default=0,
                    help="NEXT F1: feed the verifier logits as the transmitted top-K payload (e.g. 1024)")
    ap.add_argument("--k-accept", type=int, default=1, help="support size on ACCEPT rows (1 = CE; up to 1024 "
                                                            "with --target-topk: soft distillation)")
    ap.add_argument("--k-discard", type=int, default=10, help="support size on DISCARD rows (P:520; 0 = dense KL, F2)")
    ap.add_argument("--accept-loss", default="fkl", choices=["fkl", "rkl"], help="ACCEPT-row objective (F2)")
    ap.add_argument("--discard-loss", default="full", choices=["full", "restricted"],
                    help="DISCARD-row objective: full-vocab log-softmax (Q6) or SPEC's restricted softmax (F2)")
    ap.add_argument("--ntp-beta", type=float, default=0.0, help="NTP auxiliary weight with --accept-loss rkl (F2)")
    ap.add_argument("--parallel", default="vp", choices=["vp", "dp"],
                    help="N > 1: vocab-parallel weak scaling (default) or data-parallel")
    ap.add_argument("--vp", type=int, default=0, help="N > 1: vocab-parallel group size (2-D layout with --dp)")
    ap.add_argument("--dp", type=int, default=0, help="N > 1: data-parallel group count (2-D layout with --vp)")
    ap.add_argument("--comm1", action="store_true", help="N = 1: run every exchange through a 1-rank communicator")
    ap.add_argument("--eager", action="store_true", help="launch the timed steps directly instead of replaying "
                                                          "them as one captured CUDA graph")
    ap.add_argument("--optimizer", nargs="?", const="unfused", default=None, choices=["fused", "unfused"],
                    help="add the AdamW step on the fp32 master lm_head (F3): 'unfused' (default) = bwd (dW to HBM) + "
                         "aurora_adamw_step; 'fused' applies it from the dW GEMM epilogue (measured slower, DESIGN.md)")
    ap.add_argument("--workload", default="spec_loss", choices=["spec_loss", "tree_attn", "draft_layer", "full_step"],
                    help="spec_loss: the north-star hot path (default); tree_attn: NEXT F4 tree attention; "
                         "draft_layer: NEXT F4 whole draft layer (fc + decoder layer) fwd+bwd; full_step: verify + "
                         "draft layer + lm_head loss fwd/bwd (SpeculatorStep) on --config")
    ap.add_argument("--ta-config", default="ta_tree", choices=sorted(tracegen.TREE_ATTN_CONFIGS),
                    help="F4 workload (--workload tree_attn)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "tree_attn":
        run_tree_attn(args)
    elif args.workload == "draft_layer":
        run_draft_layer(args)
    elif args.workload == "full_step":
        run_full_step(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

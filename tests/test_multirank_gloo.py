"""World-size-2 gloo tests of the multi-GPU exchange plan (-m "not gpu").

The CUDA library exchanges exactly these quantities over NCCL:
  VP (vocab-parallel): C1 allgather of each rank's top-k (value, global id) list,
      merged in global (value desc, index asc) order; C3 allgather of per-row
      (m, s, u); C4 allreduce of dH.  dW stays sharded.
  DP (data-parallel over requests): C2 allreduce of (N_A, N_D); C5 allreduce of dW;
      loss allreduce.
Here two CPU processes run the per-shard maths in f64 and the real torch.distributed
collectives (gloo), and must reproduce the single-process oracle on the whole batch.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import tracegen

WS = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _vp_worker(rank, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WS)
    try:
        tr = tracegen.gen_trace(name)
        V, M = tr["V"], tr["M"]
        # shard on a non-tile boundary on purpose
        cut = V // 2 + 37
        v0, v1 = (0, cut) if rank == 0 else (cut, V)
        T = oracle.bf16_bits_to_f64(tr["T_bits"])
        k = 10
        # C1: local top-k (global ids) -> allgather -> global merge
        _, tk, _ = oracle.target_scan(T[:, v0:v1], k)
        vals = np.take_along_axis(T[:, v0:v1], tk, axis=1)
        ids = tk + v0
        gv = [torch.zeros(M, k, dtype=torch.float64) for _ in range(WS)]
        gi = [torch.zeros(M, k, dtype=torch.int64) for _ in range(WS)]
        dist.all_gather(gv, torch.from_numpy(vals))
        dist.all_gather(gi, torch.from_numpy(ids))
        allv = torch.cat(gv, 1).numpy()
        alli = torch.cat(gi, 1).numpy()
        order = np.lexsort((alli, -allv), axis=1)
        top = np.take_along_axis(alli, order, 1)[:, :k]
        am = top[:, 0]
        lab = oracle.verify(tr["draft_tokens"], tr["parents"], tr["num_nodes"], am)
        tg = oracle.row_targets(lab["row_class"], lambda m: T[m], top)
        # C3: per-row (m, s, u) over this shard -> allgather -> combine in rank order
        H64 = oracle.bf16_bits_to_f64(tr["H_bits"])
        W = tr["W_bits"]
        Z = H64 @ oracle.bf16_bits_to_f64(W[v0:v1]).T
        mx = Z.max(1)
        s = np.exp(Z - mx[:, None]).sum(1)
        u = np.zeros(M)
        for m in range(M):
            S = tg["sup_idx"][m]
            sel = (S >= v0) & (S < v1)
            u[m] = float(np.dot(tg["sup_p"][m][sel], Z[m, S[sel] - v0]))
        msu = torch.from_numpy(np.stack([mx, s, u], 1))
        g = [torch.zeros_like(msu) for _ in range(WS)]
        dist.all_gather(g, msu)
        m_all = np.stack([x.numpy()[:, 0] for x in g])
        s_all = np.stack([x.numpy()[:, 1] for x in g])
        u_all = np.stack([x.numpy()[:, 2] for x in g])
        mm = m_all.max(0)
        lse = mm + np.log((s_all * np.exp(m_all - mm)).sum(0))
        Hs = np.array([tg["H"][m] for m in range(M)])
        w = np.array([tg["w"][m] for m in range(M)])
        row_loss = np.where(lab["row_class"] == oracle.PAD, 0.0, lse - u_all.sum(0) + Hs)
        loss = float(np.dot(w, row_loss))
        # bwd on the shard with the global lse; C4 allreduce dH
        dZ = np.exp(Z - lse[:, None]) * w[:, None]
        for m in range(M):
            S = tg["sup_idx"][m]
            sel = (S >= v0) & (S < v1)
            dZ[m, S[sel] - v0] -= w[m] * tg["sup_p"][m][sel]
        dW_shard = dZ.T @ H64
        dH = torch.from_numpy(dZ @ oracle.bf16_bits_to_f64(W[v0:v1]))
        dist.all_reduce(dH)
        if rank == 0:
            q.put(dict(am=am, accept_len=lab["accept_len"], loss=loss, lse=lse, dH=dH.numpy(),
                       dW0=dW_shard, sup=[tg["sup_idx"][m] for m in range(M)]))
        else:
            q.put(dict(dW1=dW_shard))
    finally:
        dist.destroy_process_group()


def _dp_worker(rank, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WS)
    try:
        tr = tracegen.gen_trace(name)
        R, N = tr["R"], tr["N"]
        r0, r1 = (0, R // 2) if rank == 0 else (R // 2, R)
        rows = slice(r0 * (N + 1), r1 * (N + 1))
        sub = dict(tr)
        sub["draft_tokens"] = tr["draft_tokens"][r0:r1]
        sub["parents"] = None if tr["parents"] is None else tr["parents"][r0:r1]
        sub["num_nodes"] = None if tr["num_nodes"] is None else tr["num_nodes"][r0:r1]
        T = oracle.bf16_bits_to_f64(tr["T_bits"][rows])
        am, tk, _ = oracle.target_scan(T, 10)
        lab = oracle.verify(sub["draft_tokens"], sub["parents"], sub["num_nodes"], am)
        # C2: global counts -> weights
        cnt = torch.tensor([int((lab["row_class"] == 0).sum()), int((lab["row_class"] == 1).sum())])
        dist.all_reduce(cnt)
        tg = oracle.row_targets(lab["row_class"], lambda m: T[m], tk)
        na, nd = int(cnt[0]), int(cnt[1])
        for m in tg["w"]:
            c = lab["row_class"][m]
            tg["w"][m] = 1.0 / na if c == 0 else (1.0 / nd if c == 1 else 0.0)
        H64 = oracle.bf16_bits_to_f64(tr["H_bits"][rows])
        fw = oracle.loss_fwd(H64, tr["W_bits"], tg)
        bw = oracle.loss_bwd(H64, tr["W_bits"], tg, fw["lse"])
        loss = torch.tensor([fw["loss"]], dtype=torch.float64)
        dist.all_reduce(loss)
        dW = torch.from_numpy(bw["dW"])
        dist.all_reduce(dW)            # C5
        if rank == 0:
            q.put(dict(loss=float(loss.item()), dW=dW.numpy(), dH0=bw["dH"]))
    finally:
        dist.destroy_process_group()


def _spawn(fn, name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, port, name, q)) for r in range(WS)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(1 if fn is _dp_worker else WS)]
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    merged = {}
    for o in outs:
        merged.update(o)
    return merged


@pytest.mark.parametrize("name", ["small", "small_tree"])
def test_vp2_exchange_reproduces_single_rank(name):
    out = _spawn(_vp_worker, name)
    tr = tracegen.gen_trace(name)
    ref = oracle.step(tr)
    np.testing.assert_array_equal(out["am"], ref["argmax"])               # C1: bit-exact global labels
    np.testing.assert_array_equal(out["accept_len"], ref["accept_len"])
    for m in range(tr["M"]):
        np.testing.assert_array_equal(out["sup"][m], ref["targets"]["sup_idx"][m])
    np.testing.assert_allclose(out["lse"], ref["lse"], rtol=1e-12)        # C3
    assert abs(out["loss"] - ref["loss"]) <= 1e-11 * abs(ref["loss"])
    np.testing.assert_allclose(out["dH"], ref["dH"], rtol=1e-10, atol=1e-14)   # C4
    dW = np.concatenate([out["dW0"], out["dW1"]], 0)
    np.testing.assert_allclose(dW, ref["dW"], rtol=1e-10, atol=1e-14)


def test_dp2_exchange_reproduces_single_rank():
    out = _spawn(_dp_worker, "small")
    tr = tracegen.gen_trace("small")
    ref = oracle.step(tr)
    assert abs(out["loss"] - ref["loss"]) <= 1e-11 * abs(ref["loss"])      # C2 + loss allreduce
    np.testing.assert_allclose(out["dW"], ref["dW"], rtol=1e-10, atol=1e-14)   # C5
    half = (tr["R"] // 2) * (tr["N"] + 1)
    np.testing.assert_allclose(out["dH0"], ref["dH"][:half], rtol=1e-10, atol=1e-14)


def _adamw_vp_worker(rank, port, q):
    """F3 over VP shards: each rank holds rows [v0, v1) of the lm_head; the global-norm
    clip needs sum(dW^2) over ALL shards = one scalar allreduce (the library's VP
    AllReduce of norm_sq), passed in as the other shards' share (extra_sq)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WS)
    try:
        inp = tracegen.gen_adamw_inputs(4096, steps=2, grad_scale=1e-2)
        W = inp["W"].astype(np.float64).reshape(64, 64)
        v0, v1 = (0, 40) if rank == 0 else (40, 64)
        Ws, ms, vs = W[v0:v1].reshape(-1), np.zeros((v1 - v0) * 64), np.zeros((v1 - v0) * 64)
        for step, g in enumerate(inp["G"], start=1):
            gs = g.astype(np.float64).reshape(64, 64)[v0:v1].reshape(-1)
            local = torch.tensor([float(np.sum(gs * gs))], dtype=torch.float64)
            tot = local.clone()
            dist.all_reduce(tot)
            Ws, ms, vs, norm = oracle.adamw_step(Ws, ms, vs, gs, step, 1e-3, warmup_steps=0,
                                                 extra_sq=float(tot.item() - local.item()))
        q.put((rank, v0, v1, Ws, norm))
    finally:
        dist.destroy_process_group()


def test_adamw_vp_norm_exchange_matches_single_process():
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_adamw_vp_worker, args=(r, port, q)) for r in range(WS)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(WS)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    inp = tracegen.gen_adamw_inputs(4096, steps=2, grad_scale=1e-2)
    W, m, v = inp["W"].astype(np.float64), np.zeros(4096), np.zeros(4096)
    for step, g in enumerate(inp["G"], start=1):
        W, m, v, norm = oracle.adamw_step(W, m, v, g, step, 1e-3, warmup_steps=0)
    W = W.reshape(64, 64)
    for rank, v0, v1, Ws, n in res:
        assert abs(n - norm) <= 1e-12 * norm
        np.testing.assert_allclose(Ws, W[v0:v1].reshape(-1), rtol=1e-13, atol=1e-16)


def _f2_vp_worker(rank, port, q):
    """F2 (RKL + NTP on ACCEPT rows, dense KL on DISCARD rows) over two vocab shards: the
    exchanges the library makes -- C1 top lists (argmax), the T-row triples (max,
    sum e^{t-m}, sum e^{t-m} t), C3 (m, s, u, r), C4 dH -- run as gloo collectives."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WS)
    try:
        tr = tracegen.gen_trace("small_tree")
        V, M = tr["V"], tr["M"]
        cut = V // 2 + 37
        v0, v1 = (0, cut) if rank == 0 else (cut, V)
        beta = 0.5
        T = oracle.bf16_bits_to_f64(tr["T_bits"])[:, v0:v1]
        # C1 (k = 1 suffices: RKL + NTP needs only the argmax; dense discard has no support)
        loc = np.lexsort((np.arange(v1 - v0)[None, :].repeat(M, 0), -T), axis=1)[:, 0]
        cand = torch.from_numpy(np.stack([T[np.arange(M), loc], loc + v0], 1))
        g = [torch.zeros_like(cand) for _ in range(WS)]
        dist.all_gather(g, cand)
        allc = torch.stack(g).numpy()  # [rank, M, (value, id)]
        best = np.lexsort((allc[:, :, 1], -allc[:, :, 0]), axis=0)[0]
        am = allc[best, np.arange(M), 1].astype(np.int64)
        lab = oracle.verify(tr["draft_tokens"], tr["parents"], tr["num_nodes"], am)
        cls = lab["row_class"]
        na, nd = int((cls == 0).sum()), int((cls == 1).sum())
        w = np.where(cls == 0, 1.0 / na, np.where(cls == 1, 1.0 / nd, 0.0))
        # T-row triples -> global lse_t, E_p[t]
        mt = T.max(1)
        St = np.exp(T - mt[:, None]).sum(1)
        At = (np.exp(T - mt[:, None]) * T).sum(1)
        g = [torch.zeros(M, 3, dtype=torch.float64) for _ in range(WS)]
        dist.all_gather(g, torch.from_numpy(np.stack([mt, St, At], 1)))
        trip = torch.stack(g).numpy()
        mm = trip[:, :, 0].max(0)
        S = (trip[:, :, 1] * np.exp(trip[:, :, 0] - mm)).sum(0)
        Asum = (trip[:, :, 2] * np.exp(trip[:, :, 0] - mm)).sum(0)
        lse_t = mm + np.log(S)
        Hp = Asum / S - lse_t
        # C3: (m, s, u, r) per shard
        H64 = oracle.bf16_bits_to_f64(tr["H_bits"])
        Wsh = oracle.bf16_bits_to_f64(tr["W_bits"][v0:v1])
        Z = H64 @ Wsh.T
        mz = Z.max(1)
        e = np.exp(Z - mz[:, None])
        s = e.sum(1)
        r = (e * (Z - T)).sum(1)
        p = np.exp(T - lse_t[:, None])
        u = np.zeros(M)
        for m_ in range(M):
            if cls[m_] == 0 and v0 <= am[m_] < v1:
                u[m_] = beta * Z[m_, am[m_] - v0]
            elif cls[m_] == 1:
                u[m_] = float(np.dot(p[m_], Z[m_]))
        g = [torch.zeros(M, 4, dtype=torch.float64) for _ in range(WS)]
        dist.all_gather(g, torch.from_numpy(np.stack([mz, s, u, r], 1)))
        q4 = torch.stack(g).numpy()
        MM = q4[:, :, 0].max(0)
        sc = np.exp(q4[:, :, 0] - MM)
        ssum = (q4[:, :, 1] * sc).sum(0)
        R = (q4[:, :, 3] * sc).sum(0)
        U = q4[:, :, 2].sum(0)
        lse = MM + np.log(ssum)
        eqzt = R / ssum
        row_loss = np.where(cls == 0, eqzt - lse + lse_t + beta * lse - U,
                            np.where(cls == 1, lse - U + Hp, 0.0))
        loss = float(np.dot(w, row_loss))
        # bwd on the shard: dz = w (q ((z - t) - E + beta) - beta e_y) / w (q - p); C4 dH
        qz = np.exp(Z - lse[:, None])
        dZ = np.zeros_like(Z)
        for m_ in range(M):
            if cls[m_] == 0:
                dZ[m_] = qz[m_] * ((Z[m_] - T[m_]) - eqzt[m_] + beta)
                if v0 <= am[m_] < v1:
                    dZ[m_, am[m_] - v0] -= beta
            elif cls[m_] == 1:
                dZ[m_] = qz[m_] - p[m_]
            dZ[m_] *= w[m_]
        dW_shard = dZ.T @ H64
        dH = torch.from_numpy(dZ @ Wsh)
        dist.all_reduce(dH)
        q.put((rank, v0, v1, loss, dH.numpy(), dW_shard))
    finally:
        dist.destroy_process_group()


def test_f2_objectives_vp_exchange_matches_oracle():
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_f2_vp_worker, args=(r, port, q)) for r in range(WS)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=180) for _ in range(WS)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    tr = tracegen.gen_trace("small_tree")
    ref = oracle.step_variants(tr, accept_loss="rkl", ntp_beta=0.5, k_discard=0)
    for rank, v0, v1, loss, dH, dWs in res:
        assert abs(loss - ref["loss"]) <= 1e-10 * abs(ref["loss"])
        np.testing.assert_allclose(dH, ref["dH"], rtol=1e-9, atol=1e-13)
        np.testing.assert_allclose(dWs, ref["dW"][v0:v1], rtol=1e-9, atol=1e-13)

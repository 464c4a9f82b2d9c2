"""Small runs of the round-2 paths for compute-sanitizer (memcheck / racecheck / synccheck):
the staged forward + rescale backward, the TMA-ring scan, the fused AdamW kernel (k_dw_adamw),
the sharded optimizer and the multi-rank exchanges through the loopback communicator, the
A-resident dW sweep (k_dw_resident, opt-in), the one-pass tcgen05 tree attention and the draft
layer on the tcgen05 engine.

    compute-sanitizer --tool racecheck python scripts/san_r02.py [part ...]
"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import tracegen  # noqa: E402
from paper_2602_06932_b200 import aurora as A  # noqa: E402


def bf(b):
    return torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).cuda()


def spec(tr, comm=None, **kw):
    c = tr["cfg"]
    H, W = bf(tr["H_bits"]), bf(tr["W_bits"])
    draft = torch.from_numpy(tr["draft_tokens"]).cuda()
    par = None if tr["parents"] is None else torch.from_numpy(tr["parents"]).cuda()
    nn = None if tr["num_nodes"] is None else torch.from_numpy(tr["num_nodes"]).cuda()
    st = A.SpecTrainStep(c.R, c.N, c.d, c.V, comm=comm, **kw)
    st.verify(draft, bf(tr["T_bits"]), par, nn)
    st.forward(H, W)
    return st, H, W


def part_main():
    st, H, W = spec(tracegen.gen_trace("small_tree"))
    c = tracegen.CONFIGS["small_tree"]
    dH = torch.empty(c.M, c.d, device="cuda")
    dW = torch.empty(c.V, c.d, device="cuda")
    st.backward(H, W, dH, dW)                      # staged: k_dz_rescale + k_dz_support_fix
    A.aurora_set_option("dw_resident", 1)
    st.forward(H, W)
    st.backward(H, W, dH, dW)                      # k_dw_resident
    A.aurora_set_option("dw_resident", 0)
    opt = A.AdamW(W.float().reshape(-1).clone(), lr=1e-4, warmup_steps=0)
    st.forward(H, W)
    st.backward_adamw(H, W, dH, opt)               # k_dw_adamw
    torch.cuda.synchronize()
    assert int(st.status.item()) == 0


def part_multirank():
    tr = tracegen.gen_trace("small")
    c = tr["cfg"]
    comms = A.aurora_comm_create_loopback(4, 2, 2)

    def fn(rank):
        with torch.cuda.stream(torch.cuda.Stream()):
            q, v = rank // 2, rank % 2
            r0, r1 = q * c.R // 2, (q + 1) * c.R // 2
            v0, v1 = v * c.V // 2, (v + 1) * c.V // 2
            rows = slice(r0 * (c.N + 1), r1 * (c.N + 1))
            st = A.SpecTrainStep(r1 - r0, c.N, c.d, c.V, V_local=v1 - v0, vocab_offset=v0, comm=comms[rank])
            st.verify(torch.from_numpy(np.ascontiguousarray(tr["draft_tokens"][r0:r1])).cuda(),
                      bf(np.ascontiguousarray(tr["T_bits"][rows, v0:v1])), None,
                      torch.from_numpy(np.ascontiguousarray(tr["num_nodes"][r0:r1])).cuda())
            H, W = bf(np.ascontiguousarray(tr["H_bits"][rows])), bf(np.ascontiguousarray(tr["W_bits"][v0:v1]))
            st.forward(H, W)
            dH = torch.empty(st.M, c.d, device="cuda")
            dW = torch.empty(v1 - v0, c.d, device="cuda")
            st.backward(H, W, dH, dW, dp_reduce=False)
            opt = A.ShardedAdamW(W.float().reshape(-1), comms[rank], q, 2, lr=1e-4, warmup_steps=0)
            opt.step(dW.reshape(-1), W.reshape(-1))
            torch.cuda.current_stream().synchronize()

    ts = [threading.Thread(target=fn, args=(r,)) for r in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for h in comms:
        A.aurora_comm_destroy(h)


def part_attn():
    inp = tracegen.gen_tree_attn("ta_small")
    c = inp["cfg"]
    R, N1 = len(inp["requests"]), c.N + 1
    t = {k: bf(inp[k + "_bits"]) for k in ["Q", "Kt", "Vt", "Kp", "Vp", "dO"]}
    off = torch.from_numpy(inp["prefix_off"].astype(np.int32)).cuda()
    par = torch.from_numpy(inp["parents"].astype(np.int32)).cuda()
    nn = torch.from_numpy(inp["num_nodes"].astype(np.int32)).cuda()
    ta = A.TreeAttention(R, c.N, c.Hq, c.Hkv, c.dh, off, int(np.max(np.diff(inp["prefix_off"]))), parents=par,
                         num_nodes=nn)
    A.aurora_set_option("tree_fwd_tc", 2)   # the defaults: one-pass tcgen05 fwd, tcgen05 bwd
    A.aurora_set_option("tree_bwd_tc", 1)
    O = torch.empty_like(t["Q"])
    lse = torch.empty(R, N1, c.Hq, device="cuda")
    ta.forward(t["Q"], t["Kt"], t["Vt"], t["Kp"], t["Vp"], O, lse)
    dQ = torch.empty(t["Q"].shape, dtype=torch.float32, device="cuda")
    dKt, dVt, dKp, dVp = (torch.empty_like(t[k]) for k in ("Kt", "Vt", "Kp", "Vp"))
    ta.backward(t["Q"], t["Kt"], t["Vt"], t["Kp"], t["Vp"], O, lse, t["dO"], dQ, dKt, dVt, dKp, dVp)
    torch.cuda.synchronize()
    assert int(ta.status.item()) == 0


def part_scan():
    """A2 load-balanced flat scan (forced) and the k-way merge."""
    tr = tracegen.gen_trace("tiny")
    A.aurora_set_option("scan_flat", 2)
    spec(tr)
    A.aurora_set_option("scan_flat", 1)


PARTS = dict(main=part_main, multirank=part_multirank, attn=part_attn, scan=part_scan)
if __name__ == "__main__":
    A.lib()
    for name in (sys.argv[1:] or list(PARTS)):
        PARTS[name]()
    print("sanitizer round-2 paths ok")

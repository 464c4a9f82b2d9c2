"""Small runs of the newer paths for compute-sanitizer: F1 long supports (sort + long
finalize), F2 objectives (row lse of T, T-reading epilogues), F3 AdamW, graph capture."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import tracegen  # noqa: E402
from paper_2602_06932_b200 import aurora as A  # noqa: E402


def bf(b):
    return torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).cuda()


def run(tr, sparse=False, **kw):
    c = tr["cfg"]
    H, W = bf(tr["H_bits"]), bf(tr["W_bits"])
    draft = torch.from_numpy(tr["draft_tokens"]).cuda()
    par = None if tr["parents"] is None else torch.from_numpy(tr["parents"]).cuda()
    nn = None if tr["num_nodes"] is None else torch.from_numpy(tr["num_nodes"]).cuda()
    st = A.SpecTrainStep(c.R, c.N, c.d, c.V, **kw)
    if sparse:
        st.verify_topk(draft, torch.from_numpy(tr["Tk_idx"]).cuda(), bf(tr["Tk_bits"]), par, nn)
    else:
        st.verify(draft, bf(tr["T_bits"]), par, nn)
    st.forward(H, W)
    dH = torch.empty(c.M, c.d, device="cuda")
    dW = torch.empty(c.V, c.d, device="cuda")
    st.backward(H, W, dH, dW)
    torch.cuda.synchronize()
    assert int(st.status.item()) == 0
    return st, dW


A.lib()
run(tracegen.gen_trace_topk("small_tree", K_t=100), sparse=True, k_accept=40, k_discard=100)
run(tracegen.gen_trace("small"), accept_loss="rkl", ntp_beta=0.5, k_discard=0)
run(tracegen.gen_trace("small_tree"), accept_loss="rkl", k_discard=3)
inp = tracegen.gen_adamw_inputs(4096 * 33, steps=2)
Wm = torch.from_numpy(inp["W"].copy()).cuda()
opt = A.AdamW(Wm, warmup_steps=3)
Wb = torch.empty_like(Wm, dtype=torch.bfloat16)
for g in inp["G"]:
    opt.step(torch.from_numpy(g).cuda(), W_bf16=Wb)
torch.cuda.synchronize()
print("sanitizer variants ok")

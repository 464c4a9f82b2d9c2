import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import tracegen
from paper_2602_06932_b200 import aurora as A
name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
kw = dict(accept_loss="rkl", ntp_beta=0.0, k_discard=10)
tr = tracegen.gen_trace(name)
c = tr["cfg"]
bf = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).cuda()
T, H, W = bf(tr["T_bits"]), bf(tr["H_bits"]), bf(tr["W_bits"])
draft = torch.from_numpy(tr["draft_tokens"]).cuda()
st = A.SpecTrainStep(c.R, c.N, c.d, c.V, **kw)
st.verify(draft, T, None if tr["parents"] is None else torch.from_numpy(tr["parents"]).cuda(),
          None if tr["num_nodes"] is None else torch.from_numpy(tr["num_nodes"]).cuda())
torch.cuda.synchronize(); print("verify ok", st.row_lse_t[:4])
st.forward(H, W); torch.cuda.synchronize(); print("fwd ok", st.loss)
dH = torch.empty(c.M, c.d, device="cuda"); dW = torch.empty(c.V, c.d, device="cuda")
st.backward(H, W, dH, dW); torch.cuda.synchronize(); print("bwd ok")

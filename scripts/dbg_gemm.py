import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_06932_b200 import aurora as A
A.lib()
for (M, N, K) in [(128, 256, 64), (512, 1024, 1024)]:
    Am = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    Bm = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    D = torch.full((M, N), float("nan"), device="cuda")
    A.aurora_debug_gemm(False, False, Am, Bm, D, M, N, K, K, K, N)
    torch.cuda.synchronize()
    ref = Am.float() @ Bm.float().T
    print(M, N, K, "nan count", torch.isnan(D).sum().item(), "maxerr", (D - ref).abs().nan_to_num(1e9).max().item(),
          "pair_opt", A.aurora_get_option("gemm_pair"), flush=True)

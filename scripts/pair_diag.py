import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_06932_b200 import aurora as A
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_microbench import t_ms

A.lib()
M, N, K = 1792, 4096, 8192
Am = torch.randn(M, K, device="cuda").to(torch.bfloat16)
Bm = torch.randn(N, K, device="cuda").to(torch.bfloat16)
D = torch.empty(M, N, device="cuda")
for pair in (1, 2):
    A.aurora_set_option("gemm_pair", pair)
    ms = t_ms(lambda: A.aurora_debug_gemm(False, False, Am, Bm, D, M, N, K, K, K, N))
    print(json.dumps(dict(pair=pair, ms=round(ms, 4), tflops=round(2.0 * M * N * K / ms / 1e9, 1),
                          max_active_clusters=A.aurora_get_option("pair_max_active_clusters"))))
    ref = Am.float() @ Bm.float().T
    print("maxerr", (D - ref).abs().max().item())

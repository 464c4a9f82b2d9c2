"""Store-bound GEMM-engine microbenchmark over output shapes (same bytes, different
row lengths) to separate the SM-side store path from the DRAM write pattern."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_06932_b200 import aurora as A  # noqa: E402
from store_microbench import t_ms  # noqa: E402


def main():
    A.lib()
    K = int(os.environ.get("MB_K", "64"))
    for pair in (1, 2):
        A.aurora_set_option("gemm_pair", pair)
        for M, N in [(32256, 4096), (516096, 256), (129024, 1024), (8064, 16384)]:
            D = torch.empty(M, N, device="cuda")
            Am = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            Bt = torch.randn(K, N, device="cuda").to(torch.bfloat16)
            ms = t_ms(lambda: A.aurora_debug_gemm(False, True, Am, Bt, D, M, N, K, Am.stride(0), Bt.stride(0),
                                                  D.stride(0)))
            print(json.dumps(dict(pair=pair, M=M, N=N, K=K, nfast=os.environ.get("AURORA_DBG_NFAST", "0"),
                                  GBs=round(D.numel() * 4 / ms / 1e6, 1))), flush=True)
            del D, Am, Bt
            torch.cuda.empty_cache()
    A.aurora_set_option("gemm_pair", 0)


if __name__ == "__main__":
    main()

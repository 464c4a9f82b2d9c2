"""Store-bound microbenchmark of the GEMM engine's fp32 TMA-store epilogue.

D[M, N] fp32 = A B^T with small K: the output write dominates, so GB/s of D written
measures the epilogue's store pipeline against torch's write-only fill_ and copy_.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_06932_b200 import aurora as A  # noqa: E402


def t_ms(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    A.lib()
    M, N = 32256, 4096
    D = torch.empty(M, N, device="cuda")
    nbytes = D.numel() * 4
    ms = t_ms(lambda: D.fill_(1.0))
    print(json.dumps(dict(what="torch_fill", GBs=round(nbytes / ms / 1e6, 1), ms=round(ms, 4))), flush=True)
    S = torch.empty_like(D)
    ms = t_ms(lambda: D.copy_(S))
    print(json.dumps(dict(what="torch_copy_rw", GBs=round(2 * nbytes / ms / 1e6, 1), ms=round(ms, 4))), flush=True)
    del S
    for pair in (1, 2):
        A.aurora_set_option("gemm_pair", pair)
        for K in (64, 384):
            Am = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            Bt = torch.randn(K, N, device="cuda").to(torch.bfloat16)  # MN-major B like dW's H
            ms = t_ms(lambda: A.aurora_debug_gemm(False, True, Am, Bt, D, M, N, K, Am.stride(0), Bt.stride(0),
                                                  D.stride(0)))
            print(json.dumps(dict(what="umma_store", pair=pair, K=K, GBs=round(nbytes / ms / 1e6, 1),
                                  ms=round(ms, 4))), flush=True)
    A.aurora_set_option("gemm_pair", 0)


if __name__ == "__main__":
    main()

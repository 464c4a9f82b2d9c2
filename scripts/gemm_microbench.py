"""Microbenchmark of the tcgen05 GEMM engine (test hook aurora_debug_gemm) vs cuBLAS.

Times D[M,N] = A B^T for each operand-major combination at a square shape and at the
lm_head phase shapes, reporting TFLOP/s (CUDA events, warm-up, median of 10).
"""
import json
import sys
import os

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
    out = []
    shapes = [("square", 8192, 8192, 8192), ("fwd_llama", 384, 128256, 4096), ("dW_llama_chunk", 16128, 4096, 384),
              ("dH_llama_chunk", 384, 4096, 16128)]
    for name, M, N, K in shapes:
        for a_mn in (0, 1):
            for b_mn in (0, 1):
                Am = torch.randn(M, K, device="cuda").to(torch.bfloat16)
                Bm = torch.randn(N, K, device="cuda").to(torch.bfloat16)
                Ast = Am.T.contiguous() if a_mn else Am
                Bst = Bm.T.contiguous() if b_mn else Bm
                D = torch.empty(M, N, device="cuda")
                ms = t_ms(lambda: A.aurora_debug_gemm(bool(a_mn), bool(b_mn), Ast, Bst, D, M, N, K, Ast.stride(0),
                                                      Bst.stride(0), D.stride(0)))
                tf = 2.0 * M * N * K / (ms / 1e3) / 1e12
                rec = dict(shape=name, M=M, N=N, K=K, a_mn=a_mn, b_mn=b_mn, ms=round(ms, 4), tflops=round(tf, 1))
                if a_mn == 0 and b_mn == 0:
                    Dr = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
                    msb = t_ms(lambda: torch.matmul(Am, Bm.T, out=Dr))
                    rec["cublas_bf16out_tflops"] = round(2.0 * M * N * K / (msb / 1e3) / 1e12, 1)
                out.append(rec)
                print(json.dumps(rec), flush=True)
                del Am, Bm, Ast, Bst, D
                torch.cuda.empty_cache()


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def mma_bound():
    """L2-resident, MMA-bound shape: does operand major-ness cost throughput?"""
    A.lib()
    M, N, K = 1792, 4096, 8192
    for a_mn in (0, 1):
        for b_mn in (0, 1):
            Am = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            Bm = torch.randn(N, K, device="cuda").to(torch.bfloat16)
            Ast = Am.T.contiguous() if a_mn else Am
            Bst = Bm.T.contiguous() if b_mn else Bm
            D = torch.empty(M, N, device="cuda")
            ms = t_ms(lambda: A.aurora_debug_gemm(bool(a_mn), bool(b_mn), Ast, Bst, D, M, N, K, Ast.stride(0),
                                                  Bst.stride(0), D.stride(0)))
            print(json.dumps(dict(shape="mma_bound", M=M, N=N, K=K, a_mn=a_mn, b_mn=b_mn, ms=round(ms, 4),
                                  tflops=round(2.0 * M * N * K / (ms / 1e3) / 1e12, 1))), flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "mma":
    mma_bound()

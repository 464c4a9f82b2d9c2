#!/bin/bash
# Source-level ncu capture of the qwen3 dW GEMM (k_umma_gemm<2, 0, 1, 2, 256>).
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/dwprof; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; exit 1; }
timeout 600 ncu --set full --import-source on --clock-control none -k k_umma_gemm --launch-skip 2 -c 1 -o $O/prof_dw -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --eager > $O/ncu.log 2>&1; echo ncu_rc=$?; tail -2 $O/ncu.log

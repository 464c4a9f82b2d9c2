#!/bin/bash
# Targeted ncu captures (one GPU); outputs under gpurun_out/
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build_failed; tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "full_parity_small or gemm_engine" > gpurun_out/parity.log 2>&1; echo parity_rc=$?; tail -2 gpurun_out/parity.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_target_scan -c 1 -o gpurun_out/prof_scan python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_scan.log 2>&1; echo scan_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_umma_gemm -s 2 -c 2 -o gpurun_out/prof_dw_llama python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_dw.log 2>&1; echo dw_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_umma_gemm -c 4 -o gpurun_out/prof_qwen3 python bench.py --config qwen3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_q.log 2>&1; echo q_rc=$?
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2>&1; tail -1 gpurun_out/bench.json | cut -c1-900
timeout 300 python bench.py --config qwen3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_qwen3.json 2>&1; tail -1 gpurun_out/bench_qwen3.json | cut -c1-900

#!/bin/bash
# One gpurun call: bench + full-size parity + ncu evidence (outputs under gpurun_out/).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 300 python bench.py --config qwen3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_qwen3.json 2>&1; echo bq_rc=$?
tail -3 gpurun_out/bench_qwen3.json
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "llama or large" > gpurun_out/parity_full.log 2>&1; echo pf_rc=$?
tail -15 gpurun_out/parity_full.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_umma_gemm -s 13 -c 4 -o gpurun_out/prof_gemm python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
bash scripts/gpu_sanitize2.sh
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo gpu_tests_rc=$?; tail -4 gpurun_out/gpu_tests.log
timeout 400 python bench.py > gpurun_out/b_default.json 2> gpurun_out/b_default.err; echo bench_rc=$?; tail -1 gpurun_out/b_default.json | cut -c1-300
timeout 600 ncu --set full --clock-control none -k regex:k_target_scan -c 1 -o gpurun_out/prof_r3_scan python bench.py --steps 1 --warmup 3 --no-cpu-baseline --eager > gpurun_out/ncu_scan.log 2>&1; echo ncu_s_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --eager > gpurun_out/ncu_launches.log 2>&1; echo ncu_l_rc=$?

#!/bin/bash
# Full validation + evidence round (one GPU).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build_failed; tail -20 gpurun_out/build.log; exit 1; }
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo gpu_tests_rc=$?; tail -4 gpurun_out/gpu_tests.log
timeout 400 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?; tail -1 gpurun_out/bench_default.json | cut -c1-3000
timeout 400 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo ref_rc=$?; tail -1 gpurun_out/bench_ref.json | cut -c1-600
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo ncu_l_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_umma_gemm -s 14 -c 4 -o gpurun_out/prof_final python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_final.log 2>&1; echo ncu_f_rc=$?
timeout 600 ncu --set full --clock-control none -k regex:k_target_scan -c 1 -o gpurun_out/prof_scan_final python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_scan_final.log 2>&1; echo ncu_s_rc=$?
ls -la gpurun_out | tail -20

#!/bin/bash
# Full validation + evidence: GPU suite, bench lines per workload/variant, ncu captures.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build_failed; tail -20 gpurun_out/build.log; exit 1; }
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo gpu_tests_rc=$?; tail -4 gpurun_out/gpu_tests.log
b() { local name=$1; shift; timeout 400 python bench.py "$@" > gpurun_out/b_$name.json 2> gpurun_out/b_$name.err; echo "bench $name rc=$?"; tail -1 gpurun_out/b_$name.json | cut -c1-400; }
b default
b qwen3 --config qwen3 --steps 10 --warmup 3 --no-cpu-baseline
b minimax --config minimax --steps 5 --warmup 3 --no-cpu-baseline
b f1 --config llama_d32k --target-topk 1024 --k-accept 1024 --k-discard 1024 --no-cpu-baseline
b f1_llama --target-topk 1024 --no-cpu-baseline
b f2 --accept-loss rkl --ntp-beta 0.5 --k-discard 0 --no-cpu-baseline
b f3 --optimizer --no-cpu-baseline
timeout 400 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/b_ref.json 2>&1; echo ref_rc=$?; tail -1 gpurun_out/b_ref.json | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo ncu_l_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_umma_gemm -s 4 -c 4 -o gpurun_out/prof_r2_gemm python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_gemm.log 2>&1; echo ncu_g_rc=$?
timeout 600 ncu --set full --clock-control none -k regex:k_target_scan -c 1 -o gpurun_out/prof_r2_scan python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_scan.log 2>&1; echo ncu_s_rc=$?
timeout 600 ncu --set full --clock-control none -k regex:k_adamw -c 1 -o gpurun_out/prof_r2_adamw python bench.py --steps 1 --warmup 1 --no-cpu-baseline --optimizer > gpurun_out/ncu_adamw.log 2>&1; echo ncu_a_rc=$?
ls gpurun_out | tail -30

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/v2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/v2/build.log 2>&1 || { echo build_failed; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v2/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/v2/smoke.log | cut -c1-250
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/v2/gpu_tests.log 2>&1; echo gpu_tests_rc=$?; tail -2 gpurun_out/v2/gpu_tests.log
timeout 400 python bench.py > gpurun_out/v2/b_llama.json 2> gpurun_out/v2/b_llama.err; echo bench_rc=$?; tail -1 gpurun_out/v2/b_llama.json | cut -c1-200

#!/bin/bash
# F1 validation: topk ingest parity, full GPU suite, topk bench.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build_failed; tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "topk" > gpurun_out/f1_tests.log 2>&1; echo f1_rc=$?; tail -15 gpurun_out/f1_tests.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo gpu_tests_rc=$?; tail -8 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --target-topk 1024 --no-cpu-baseline > gpurun_out/bench_topk.json 2> gpurun_out/bench_topk.err; echo btk_rc=$?; tail -1 gpurun_out/bench_topk.json | cut -c1-2500; tail -3 gpurun_out/bench_topk.err
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?; tail -1 gpurun_out/bench.json | cut -c1-2500; tail -3 gpurun_out/bench.err

#!/bin/bash
# Re-entry verification: GPU tests, smoke, default bench, comm1 bench, every workload.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo gpu_tests_rc=$?; tail -4 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/b_default.json 2> gpurun_out/b_default.err; echo bench_rc=$?; tail -1 gpurun_out/b_default.json | cut -c1-400
timeout 400 python bench.py --comm1 --no-cpu-baseline > gpurun_out/b_comm1.json 2> gpurun_out/b_comm1.err; echo comm1_rc=$?; tail -1 gpurun_out/b_comm1.json | cut -c1-300
for c in qwen3 minimax tree; do
  timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; echo ${c}_rc=$?; tail -1 gpurun_out/b_$c.json | cut -c1-300
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err; echo ref_rc=$?; tail -1 gpurun_out/b_ref.json | cut -c1-300

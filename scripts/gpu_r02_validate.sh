#!/bin/bash
# Validation of the committed state: build, smoke, every GPU test, default bench, ta_tree.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/validate; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log | cut -c1-200
timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo gpu_tests_rc=$?; grep -E "passed|failed" $O/gpu_tests.log | tail -1; grep -E "^FAILED" $O/gpu_tests.log | head
run() { name=$1; shift; timeout 600 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | cut -c1-200; }
run qwen3
run ta_tree --workload tree_attn --ta-config ta_tree --no-cpu-baseline

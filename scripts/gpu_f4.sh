#!/bin/bash
# F4 tree attention: parity tests, memcheck on the small case, bench lines.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -m paper_2602_06932_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_tree_attn.py -q -x > gpurun_out/f4_tests.log 2>&1; echo f4_tests_rc=$?; tail -30 gpurun_out/f4_tests.log
timeout 300 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_tree_attn.py -q -x -k "parity and ta_small" > gpurun_out/f4_memcheck.log 2>&1; echo memcheck_rc=$?; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/f4_memcheck.log | tail -3
for c in ta_tree ta_llama; do
  timeout 400 python bench.py --workload tree_attn --ta-config $c > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; echo ${c}_rc=$?; tail -1 gpurun_out/b_$c.json | cut -c1-1500; tail -3 gpurun_out/b_$c.err
done

#!/bin/bash
# compute-sanitizer over the F4 tree-attention kernels (every fwd/bwd variant) on the small case.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python -m pytest tests/test_gpu_tree_attn.py -q -x -k "parity and ta_small" > gpurun_out/sanitizer/r01_f4_$tool.log 2>&1
  echo ${tool}_rc=$?; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitizer/r01_f4_$tool.log | tail -3
done

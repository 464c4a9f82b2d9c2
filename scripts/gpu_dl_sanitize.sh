#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/sanitizer
python -m paper_2602_06932_b200.build > /dev/null
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool python -m pytest tests/test_gpu_draft_layer.py tests/test_gpu_tree_attn.py -q -x -k "draft_layer or rope" > gpurun_out/sanitizer/r01_f4_layer_$tool.log 2>&1
  echo ${tool}_rc=$?; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitizer/r01_f4_layer_$tool.log | tail -3
done

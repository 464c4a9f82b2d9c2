#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -m paper_2602_06932_b200.build > /dev/null
timeout 600 python -m pytest tests/test_gpu_draft_layer.py -q -x -s > gpurun_out/dl_tests.log 2>&1; echo dl_rc=$?; tail -30 gpurun_out/dl_tests.log

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/dl
python -m paper_2602_06932_b200.build > /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dl/launches_dl_tree.csv python bench.py --workload draft_layer --ta-config ta_tree --steps 1 --warmup 1 --eager > gpurun_out/dl/ncu_dl.log 2>&1; echo ncu_rc=$?; tail -2 gpurun_out/dl/ncu_dl.log | cut -c1-200

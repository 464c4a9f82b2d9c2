#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -m paper_2602_06932_b200.build > /dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ta_ -c 4 -o gpurun_out/prof_ta_tree -f python bench.py --workload tree_attn --ta-config ta_tree --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_ta.log 2>&1; echo ncu_rc=$?; tail -5 gpurun_out/ncu_ta.log

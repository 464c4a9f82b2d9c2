#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -m paper_2602_06932_b200.build > /dev/null
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_ta_fwd -c 1 -o gpurun_out/prof_ta_tc -f python bench.py --workload tree_attn --ta-config ta_tree --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_ta_tc.log 2>&1; echo ncu_rc=$?

#!/bin/bash
# Closing F4 evidence after the last backward changes: bench lines (attention, draft layer, whole
# step, qwen3 headline) and ncu --set full of the tree-attention kernels at ta_tree.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/final4; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log | cut -c1-120
run() { name=$1; shift; timeout 600 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | cut -c1-160; }
run qwen3
run ta_tree --workload tree_attn --ta-config ta_tree
run ta_llama --workload tree_attn --ta-config ta_llama --no-cpu-baseline
run dl_tree --workload draft_layer --ta-config ta_tree --no-cpu-baseline
run dl_llama --workload draft_layer --ta-config ta_llama --no-cpu-baseline
run fs_llama --workload full_step --config llama --no-cpu-baseline
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_ta_" -c 2 -o $O/prof_ta_tree -f python bench.py --workload tree_attn --ta-config ta_tree --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_ta.log 2>&1; echo ncu_ta_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_ta_tree.csv python bench.py --workload tree_attn --ta-config ta_tree --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_l.log 2>&1; echo ncu_l_rc=$?

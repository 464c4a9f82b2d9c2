#!/bin/bash
# F4 closing evidence: bench lines (ta_tree, ta_llama), ncu --set full of the F4 kernels.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/f4final
O=gpurun_out/f4final
python -m paper_2602_06932_b200.build > /dev/null
for c in ta_tree ta_llama; do
  timeout 500 python bench.py --workload tree_attn --ta-config $c > $O/b_$c.json 2> $O/b_$c.err; echo ${c}_rc=$?; tail -1 $O/b_$c.json | cut -c1-200
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ta_ -c 3 -o $O/prof_ta_tree -f python bench.py --workload tree_attn --ta-config ta_tree --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_ta.log 2>&1; echo ncu_ta_rc=$?

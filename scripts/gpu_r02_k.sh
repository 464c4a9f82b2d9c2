#!/bin/bash
# F3 fused AdamW entry shapes 0 / 1 / 2 (parity + bench); ncu --set full of the tcgen05 one-pass
# tree-attention forward (tree_fwd_tc=2) at ta_tree with source lines.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02k; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 400 python -m pytest tests/test_gpu_optim.py -q -x > $O/t_optim.log 2>&1; echo optim_rc=$?; tail -2 $O/t_optim.log; grep -E "^E " $O/t_optim.log | head -5
run() { name=$1; shift; timeout 300 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | cut -c1-120; tail -2 $O/b_$name.err; }
for qe in 0 1 2 0 1 2; do AURORA_DW_ADAMW_QE=$qe run f3_qe$qe --config llama --optimizer fused --no-cpu-baseline; done
AURORA_TREE_FWD_TC=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_ta_fwd_tc2" -c 1 -o $O/prof_tc2 -f python bench.py --workload tree_attn --ta-config ta_tree --steps 1 --warmup 1 --no-cpu-baseline --eager > $O/ncu2.log 2>&1; echo ncu2_rc=$?

#!/bin/bash
# tcgen05 tree attention: one-pass fwd (tc3 deep rings) and the tcgen05 backward; tests under a
# short timeout first (hang detection), then benches of every combination.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02attn; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 180 python -m pytest tests/test_gpu_tree_attn.py -q -x -k "tc3 and ta_small" > $O/t_tc3.log 2>&1; echo tc3_rc=$?; tail -2 $O/t_tc3.log
timeout 180 python -m pytest tests/test_gpu_tree_attn.py -q -x -k "tcgen05_backward and ta_small and 0" > $O/t_btc.log 2>&1; echo btc_rc=$?; tail -2 $O/t_btc.log; grep -E "^E " $O/t_btc.log | head -5
timeout 900 python -m pytest tests/test_gpu_tree_attn.py -q > $O/t_all.log 2>&1; echo tall_rc=$?; grep -E "passed|failed" $O/t_all.log | tail -1; grep -E "^FAILED" $O/t_all.log | head
run() { name=$1; shift; timeout 300 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | cut -c1-120; tail -2 $O/b_$name.err; }
for f in 0 3; do for b in 0 1; do
  AURORA_TREE_FWD_TC=$f AURORA_TREE_BWD_TC=$b run tree_f${f}_b${b} --workload tree_attn --ta-config ta_tree --no-cpu-baseline
  AURORA_TREE_FWD_TC=$f AURORA_TREE_BWD_TC=$b run llama_f${f}_b${b} --workload tree_attn --ta-config ta_llama --no-cpu-baseline
done; done

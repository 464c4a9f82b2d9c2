#!/bin/bash
# Session-3 state check: build, smoke, tree-attention tests, the fwd/bwd tcgen05 matrix, qwen3 bench.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/s3a; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log | cut -c1-200
timeout 900 python -m pytest tests/test_gpu_tree_attn.py -q > $O/t_attn.log 2>&1; echo tattn_rc=$?; grep -E "passed|failed" $O/t_attn.log | tail -1; grep -E "^FAILED" $O/t_attn.log | head
run() { name=$1; shift; timeout 300 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | cut -c1-140; tail -1 $O/b_$name.err | cut -c1-200; }
run qwen3 --no-cpu-baseline
for f in 0 3 4 5; do for b in 0 1; do
  AURORA_TREE_FWD_TC=$f AURORA_TREE_BWD_TC=$b run tree_f${f}_b${b} --workload tree_attn --ta-config ta_tree --no-cpu-baseline
  AURORA_TREE_FWD_TC=$f AURORA_TREE_BWD_TC=$b run llama_f${f}_b${b} --workload tree_attn --ta-config ta_llama --no-cpu-baseline
done; done

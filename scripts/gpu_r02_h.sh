#!/bin/bash
# Round-2 pass H: vectorised draft-layer elementwise kernels, Gram-form fused-optimizer norm,
# tcgen05 one-pass attention fix; tests; benches; compute-sanitizer on the round-2 paths.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02h; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_tree_attn.py -q -x -k "tc2" > $O/t_tc2.log 2>&1; echo tc2_rc=$?; tail -2 $O/t_tc2.log
timeout 1200 python -m pytest tests/test_gpu_draft_layer.py tests/test_gpu_optim.py tests/test_gpu_parity.py -q > $O/t.log 2>&1; echo t_rc=$?; grep -E "passed|failed" $O/t.log | tail -2; grep -E "^FAILED" $O/t.log | head
run() { name=$1; shift; timeout 300 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | cut -c1-150; tail -2 $O/b_$name.err; }
run dl_tree --workload draft_layer --ta-config ta_tree --no-cpu-baseline
run dl_llama --workload draft_layer --ta-config ta_llama --no-cpu-baseline
AURORA_TREE_FWD_TC=2 run ta_tree_tc2 --workload tree_attn --ta-config ta_tree --no-cpu-baseline
run llama_fused --config llama --optimizer fused --no-cpu-baseline
run llama_unfused --config llama --optimizer unfused --no-cpu-baseline
for tool in memcheck racecheck; do
  for part in main multirank attn; do
    timeout 600 compute-sanitizer --tool $tool --target-processes all python scripts/san_r02.py $part > $O/san_${tool}_${part}.log 2>&1; echo san_${tool}_${part}_rc=$?; tail -2 $O/san_${tool}_${part}.log
  done
done

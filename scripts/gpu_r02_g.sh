#!/bin/bash
# Round-2 pass G: tcgen05 one-pass attention (divergence fix) first under a short timeout; tests;
# attention and draft-layer benches; draft-layer launch list.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02g; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 240 python -m pytest tests/test_gpu_tree_attn.py -q -x -k "tc2" > $O/t_tc2.log 2>&1; echo tc2_rc=$?; tail -3 $O/t_tc2.log
timeout 1500 python -m pytest tests/test_gpu_tree_attn.py tests/test_gpu_optim.py tests/test_gpu_draft_layer.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -k "not tc2 or full_size" > $O/t.log 2>&1; echo t_rc=$?; grep -E "passed|failed" $O/t.log | tail -2; grep -E "^FAILED" $O/t.log | head
run() { name=$1; shift; timeout 300 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | cut -c1-150; tail -2 $O/b_$name.err; }
AURORA_TREE_FWD_TC=2 run ta_tree_tc2 --workload tree_attn --ta-config ta_tree --no-cpu-baseline
AURORA_TREE_FWD_TC=2 run ta_llama_tc2 --workload tree_attn --ta-config ta_llama --no-cpu-baseline
run dl_tree --workload draft_layer --ta-config ta_tree --no-cpu-baseline
run dl_llama --workload draft_layer --ta-config ta_llama --no-cpu-baseline
run llama_fused --config llama --optimizer fused --no-cpu-baseline
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_dl_tree.csv python bench.py --workload draft_layer --ta-config ta_tree --steps 1 --warmup 1 --no-cpu-baseline --eager > $O/ncu_dl.log 2>&1; echo ncu_dl_rc=$?

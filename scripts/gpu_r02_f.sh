#!/bin/bash
# Round-2 pass F: per-warp ring scan, fused AdamW fix, tcgen05 one-pass attention; draft-layer
# launch list (engine GEMMs vs round-1 cuBLAS).
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log | cut -c1-200
timeout 1200 python -m pytest tests/test_gpu_optim.py tests/test_gpu_tree_attn.py tests/test_gpu_fullsize.py -q > $O/t.log 2>&1; echo t_rc=$?; grep -E "passed|failed" $O/t.log | tail -2; grep -E "^FAILED" $O/t.log | head
run() { name=$1; shift; timeout 600 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | cut -c1-150; tail -2 $O/b_$name.err; }
run qwen3 --no-cpu-baseline
run llama --config llama --no-cpu-baseline
run llama_fused --config llama --optimizer fused --no-cpu-baseline
AURORA_TREE_FWD_TC=0 run ta_tree_sync --workload tree_attn --ta-config ta_tree --no-cpu-baseline
AURORA_TREE_FWD_TC=2 run ta_tree_tc2 --workload tree_attn --ta-config ta_tree --no-cpu-baseline
AURORA_TREE_FWD_TC=0 run ta_llama_sync --workload tree_attn --ta-config ta_llama --no-cpu-baseline
AURORA_TREE_FWD_TC=2 run ta_llama_tc2 --workload tree_attn --ta-config ta_llama --no-cpu-baseline
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_dl_tree.csv python bench.py --workload draft_layer --ta-config ta_tree --steps 1 --warmup 1 --no-cpu-baseline --eager > $O/ncu_dl.log 2>&1; echo ncu_dl_rc=$?

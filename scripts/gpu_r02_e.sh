#!/bin/bash
# Round-2 pass E: scan warm start; fused AdamW 32-column entries; draft layer on the tcgen05
# engine with the final norm; all GPU tests; benches; ncu.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02e; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -2 $O/smoke.log | cut -c1-300
timeout 2400 python -m pytest tests -m gpu -q > $O/t.log 2>&1; echo t_rc=$?; grep -E "passed|failed" $O/t.log | tail -3; grep -E "^FAILED" $O/t.log | head -20
run() { name=$1; shift; timeout 600 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | cut -c1-200; tail -3 $O/b_$name.err; }
run qwen3 --no-cpu-baseline
run llama --config llama --no-cpu-baseline
run llama_fused --config llama --optimizer fused --no-cpu-baseline
run dl_tree --workload draft_layer --ta-config ta_tree --no-cpu-baseline
run dl_llama --workload draft_layer --ta-config ta_llama --no-cpu-baseline
run fs_llama --workload full_step --config llama --no-cpu-baseline
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_dw_adamw|k_target_scan_ring" -c 2 -o $O/prof_adamw_scan -f python bench.py --config llama --optimizer fused --steps 1 --warmup 1 --no-cpu-baseline --eager > $O/ncu1.log 2>&1; echo ncu1_rc=$?

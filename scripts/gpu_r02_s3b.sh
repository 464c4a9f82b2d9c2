#!/bin/bash
# Flat scan (parity + timing) and ncu --set full of the tree-attention kernels at ta_tree.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/s3b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "scan" > $O/t_scan.log 2>&1; echo tscan_rc=$?; tail -2 $O/t_scan.log; grep -E "^(FAILED|E )" $O/t_scan.log | head -5
run() { name=$1; shift; timeout 240 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('phases_ms_per_step'))" 2>&1 | cut -c1-300; }
run qwen3_flat --no-cpu-baseline
AURORA_SCAN_FLAT=0 run qwen3_seg --no-cpu-baseline
AURORA_SCAN_FLAT_CTAS=2 run qwen3_flat2 --no-cpu-baseline
run llama_flat --config llama --no-cpu-baseline
AURORA_SCAN_FLAT=0 run llama_seg --config llama --no-cpu-baseline
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_target_scan" -c 1 -o $O/prof_scan -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --eager > $O/ncu_scan.log 2>&1; echo ncu_scan_rc=$?
timeout 400 ncu --set full --import-source on --clock-control none -k regex:"k_ta_fwd|k_ta_bwd_fused" -c 2 -o $O/prof_ta_sync -f python bench.py --workload tree_attn --ta-config ta_tree --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_ta_sync.log 2>&1; echo ncu_ta_sync_rc=$?
AURORA_TREE_FWD_TC=3 AURORA_TREE_BWD_TC=1 timeout 400 ncu --set full --import-source on --clock-control none -k regex:"k_ta_fwd_tc2|k_ta_bwd_tc" -c 2 -o $O/prof_ta_tc -f python bench.py --workload tree_attn --ta-config ta_tree --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_ta_tc.log 2>&1; echo ncu_ta_tc_rc=$?
timeout 600 python -m pytest tests/test_gpu_tree_attn.py -q -x > $O/t_attn.log 2>&1; echo tattn_rc=$?; tail -2 $O/t_attn.log; grep -E "^(FAILED|E )" $O/t_attn.log | head -5

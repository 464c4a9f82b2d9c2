#!/bin/bash
# Rewritten tcgen05 forward softmax + double-buffered flat scan: tests then timings.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/s3c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_tree_attn.py -q -x -k "parity and tc" > $O/t_attn.log 2>&1; echo tattn_rc=$?; tail -2 $O/t_attn.log; grep -E "^(FAILED|E )" $O/t_attn.log | head -5
timeout 400 python -m pytest tests/test_gpu_fullsize.py -q -x -k "scan" > $O/t_scan.log 2>&1; echo tscan_rc=$?; tail -1 $O/t_scan.log; grep -E "^(FAILED|E )" $O/t_scan.log | head -5
run() { name=$1; shift; timeout 240 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('phases_ms_per_step'))" 2>&1 | cut -c1-300; }
for f in 0 2 3; do
  AURORA_TREE_FWD_TC=$f run tree_f$f --workload tree_attn --ta-config ta_tree --no-cpu-baseline
  AURORA_TREE_FWD_TC=$f run llama_f$f --workload tree_attn --ta-config ta_llama --no-cpu-baseline
done
run qwen3_flat --no-cpu-baseline
AURORA_SCAN_FLAT=0 run qwen3_seg --no-cpu-baseline
run llama_flat --config llama --no-cpu-baseline
AURORA_SCAN_FLAT=0 run llama_seg --config llama --no-cpu-baseline
AURORA_TREE_FWD_TC=2 timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_ta_fwd_tc2" -c 1 -o $O/prof_tc2 -f python bench.py --workload tree_attn --ta-config ta_tree --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_tc2.log 2>&1; echo ncu_tc2_rc=$?
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_target_scan" -c 1 -o $O/prof_scan -f python bench.py --config llama --steps 1 --warmup 1 --no-cpu-baseline --eager > $O/ncu_scan.log 2>&1; echo ncu_scan_rc=$?

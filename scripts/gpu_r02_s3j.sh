#!/bin/bash
# Flat scan software-pipelined (two batches in flight per warp): parity + timings.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/s3j; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 400 python -m pytest tests/test_gpu_fullsize.py -q -x -k "scan" > $O/t_scan.log 2>&1; echo tscan_rc=$?; tail -1 $O/t_scan.log; grep -E "^(FAILED|E )" $O/t_scan.log | head -5
run() { name=$1; shift; timeout 240 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('phases_ms_per_step'))" 2>&1 | cut -c1-300; }
AURORA_SCAN_FLAT=2 run qwen3_2 --no-cpu-baseline
AURORA_SCAN_FLAT=2 run llama_2 --config llama --no-cpu-baseline
AURORA_SCAN_FLAT=2 AURORA_SCAN_FLAT_CTAS=3 run llama_2c3 --config llama --no-cpu-baseline
AURORA_SCAN_FLAT=0 run llama_0 --config llama --no-cpu-baseline
AURORA_SCAN_FLAT=0 run qwen3_0 --no-cpu-baseline
AURORA_SCAN_FLAT=2 timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_target_scan|k_topk_merge" -c 2 -o $O/prof_scan_llama -f python bench.py --config llama --steps 1 --warmup 1 --no-cpu-baseline --eager > $O/ncu_scan.log 2>&1; echo ncu_scan_rc=$?

#!/bin/bash
# Round-2 pass D: TMA-ring scan + LSU write-back fused AdamW; tests; bench; ncu of both.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_optim.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py -q -x > $O/t.log 2>&1; echo t_rc=$?; tail -5 $O/t.log
run() { name=$1; shift; timeout 600 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | cut -c1-200; tail -3 $O/b_$name.err; }
run qwen3 --no-cpu-baseline
run llama --config llama --no-cpu-baseline
run llama_fused --config llama --optimizer fused --no-cpu-baseline
run llama_unfused --config llama --optimizer unfused --no-cpu-baseline
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_dw_adamw|k_target_scan_ring" -c 2 -o $O/prof_adamw_scan -f python bench.py --config llama --optimizer fused --steps 1 --warmup 1 --no-cpu-baseline --eager > $O/ncu1.log 2>&1; echo ncu1_rc=$?

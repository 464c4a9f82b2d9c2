#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02i; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_optim.py tests/test_gpu_parity.py -q -k "adamw or fused or bf16_dw or gram" > $O/t.log 2>&1; echo t_rc=$?; grep -E "passed|failed" $O/t.log | tail -2; grep -E "^FAILED" $O/t.log | head
run() { name=$1; shift; timeout 300 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | cut -c1-150; tail -2 $O/b_$name.err; }
run llama_fused --config llama --optimizer fused --no-cpu-baseline
AURORA_SERIAL_BWD=0 run qwen3_conc --no-cpu-baseline
AURORA_SERIAL_BWD=0 run llama_conc --config llama --no-cpu-baseline
run qwen3 --no-cpu-baseline
timeout 400 ncu --set full --import-source on --clock-control none -k regex:"k_dw_adamw" -c 1 -o $O/prof_adamw -f python bench.py --config llama --optimizer fused --steps 1 --warmup 1 --no-cpu-baseline --eager > $O/ncu1.log 2>&1; echo ncu1_rc=$?

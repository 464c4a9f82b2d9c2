#!/bin/bash
# Round-2 pass C: staged forward (no recompute GEMM) — parity, multirank, optimizer tests;
# qwen3 / llama bench; ncu of the fused AdamW kernel and of the staged fwd + rescale.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -2 $O/smoke.log | cut -c1-300
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_optim.py tests/test_gpu_multirank.py tests/test_gpu_fullsize.py -q -x > $O/t.log 2>&1; echo t_rc=$?; tail -15 $O/t.log
run() { name=$1; shift; timeout 600 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | cut -c1-300; tail -3 $O/b_$name.err; }
run qwen3 --no-cpu-baseline
run llama --config llama --no-cpu-baseline
run llama_fused --config llama --optimizer fused --no-cpu-baseline
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dw_adamw -c 1 -o $O/prof_dw_adamw -f python bench.py --config llama --optimizer fused --steps 1 --warmup 1 --no-cpu-baseline --eager > $O/ncu1.log 2>&1; echo ncu1_rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_umma_gemm|k_dz_rescale" -c 4 -o $O/prof_stage -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --eager > $O/ncu2.log 2>&1; echo ncu2_rc=$?

#!/bin/bash
# Round-2 pass B: new GPU tests (full-size qwen3, multi-rank loopback, optimizer), fused vs
# unfused optimizer bench at llama, default bench.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_optim.py tests/test_gpu_multirank.py -q -x > $O/t_optim_multi.log 2>&1; echo t1_rc=$?; tail -15 $O/t_optim_multi.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > $O/t_full.log 2>&1; echo t2_rc=$?; tail -15 $O/t_full.log
run() { name=$1; shift; timeout 600 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | cut -c1-400; tail -3 $O/b_$name.err; }
run llama_opt_unfused --config llama --optimizer unfused --no-cpu-baseline
run llama_opt_fused --config llama --optimizer fused --no-cpu-baseline
run qwen3 --no-cpu-baseline

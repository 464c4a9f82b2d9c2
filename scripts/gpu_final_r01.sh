#!/bin/bash
# Round-1 closing evidence: build, smoke, every GPU test, bench lines per workload, reference arm,
# ncu launch list of the default bench, ncu --set full of the F4 kernels.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/final
O=gpurun_out/final
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log | cut -c1-300
timeout 1800 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo gpu_tests_rc=$?; tail -2 $O/gpu_tests.log
run() { name=$1; shift; timeout 500 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | cut -c1-200; }
run llama
run qwen3 --config qwen3 --no-cpu-baseline
run minimax --config minimax --no-cpu-baseline
run tree --config tree --no-cpu-baseline
run f1_d32k --config llama_d32k --target-topk 1024 --k-accept 1024 --k-discard 1024 --no-cpu-baseline
run f1_llama --target-topk 1024 --no-cpu-baseline
run f2 --accept-loss rkl --ntp-beta 0.5 --k-discard 0 --no-cpu-baseline
run f3 --optimizer --no-cpu-baseline
run comm1 --comm1 --no-cpu-baseline
run ta_tree --workload tree_attn --ta-config ta_tree
run ta_llama --workload tree_attn --ta-config ta_llama
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > $O/b_ref.json 2> $O/b_ref.err; echo ref_rc=$?; tail -1 $O/b_ref.json | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_llama.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --eager > $O/ncu_launches.log 2>&1; echo ncu_l_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ta_ -c 3 -o $O/prof_ta_tree -f python bench.py --workload tree_attn --ta-config ta_tree --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_ta.log 2>&1; echo ncu_ta_rc=$?
ls $O | head -50

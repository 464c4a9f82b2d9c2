#!/bin/bash
# Round-2 closing evidence pass: build, smoke, every GPU test, the bench line of every workload,
# the reference arm, the ncu launch list of the default bench (qwen3) + ncu --set full of its
# kernels, the tree-attention kernels (ncu --set full) and the draft-layer launch list, and
# compute-sanitizer on the new default paths.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/final3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log | cut -c1-200
timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo gpu_tests_rc=$?; grep -E "passed|failed" $O/gpu_tests.log | tail -1; grep -E "^FAILED" $O/gpu_tests.log | head
run() { name=$1; shift; timeout 600 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | cut -c1-160; }
run qwen3
run llama --config llama --no-cpu-baseline
run minimax --config minimax --no-cpu-baseline
run tree --config tree --no-cpu-baseline
run f1_d32k --config llama_d32k --target-topk 1024 --k-accept 1024 --k-discard 1024 --no-cpu-baseline
run f2_rkl --config llama --accept-loss rkl --ntp-beta 0.5 --k-discard 0 --no-cpu-baseline
run f2_restricted --config llama --discard-loss restricted --no-cpu-baseline
run f3_fused --config llama --optimizer fused --no-cpu-baseline
run f3_unfused --config llama --optimizer unfused --no-cpu-baseline
run comm1 --comm1 --no-cpu-baseline
run ta_tree --workload tree_attn --ta-config ta_tree
run ta_llama --workload tree_attn --ta-config ta_llama --no-cpu-baseline
run dl_tree --workload draft_layer --ta-config ta_tree --no-cpu-baseline
run dl_llama --workload draft_layer --ta-config ta_llama --no-cpu-baseline
run fs_llama --workload full_step --config llama --no-cpu-baseline
timeout 500 python bench.py --impl reference --steps 3 --warmup 3 > $O/b_ref.json 2> $O/b_ref.err; echo ref_rc=$?; tail -1 $O/b_ref.json | cut -c1-160
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_qwen3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --eager > $O/ncu_launches.log 2>&1; echo ncu_l_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_umma_gemm|k_dz_rescale|k_target_scan|k_topk_merge|k_row_combine|k_reduce_partials" -c 9 -o $O/prof_qwen3 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --eager > $O/ncu_full.log 2>&1; echo ncu_full_rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_ta_" -c 4 -o $O/prof_ta_tree -f python bench.py --workload tree_attn --ta-config ta_tree --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_ta.log 2>&1; echo ncu_ta_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_dl_tree.csv python bench.py --workload draft_layer --ta-config ta_tree --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_dl.log 2>&1; echo ncu_dl_rc=$?
for t in memcheck racecheck; do timeout 600 compute-sanitizer --tool $t python scripts/san_r02.py attn scan > $O/san_${t}_attn_scan.log 2>&1; echo san_${t}_rc=$?; tail -2 $O/san_${t}_attn_scan.log; done

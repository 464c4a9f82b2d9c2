#!/bin/bash
# Closing lm_head evidence (final build): qwen3 launch list + ncu --set full of the step's kernels.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/final5; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_qwen3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --eager > $O/ncu_launches.log 2>&1; echo ncu_l_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_umma_gemm|k_dz_rescale|k_target_scan|k_topk_merge|k_row_combine|k_reduce_partials|k_splitk_reduce" -c 9 -o $O/prof_qwen3 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --eager > $O/ncu_full.log 2>&1; echo ncu_full_rc=$?

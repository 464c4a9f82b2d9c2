cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_umma_gemm -s 3 -c 1 -o gpurun_out/prof_pair python scripts/pair_diag.py > gpurun_out/ncu_pair.log 2>&1; echo rc=$?
timeout 300 ncu --set full --clock-control none -k regex:k_umma_gemm -s 23 -c 1 -o gpurun_out/prof_pair2 python scripts/pair_diag.py > gpurun_out/ncu_pair2.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu_pair2.log

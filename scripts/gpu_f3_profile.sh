#!/bin/bash
# F3 fused AdamW kernel: source-level ncu capture (stall reasons) at llama.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/s3l; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_dw_adamw" -c 1 -o $O/prof_dwadamw -f python bench.py --config llama --optimizer fused --steps 1 --warmup 1 --no-cpu-baseline --eager > $O/ncu.log 2>&1; echo ncu_rc=$?; tail -3 $O/ncu.log

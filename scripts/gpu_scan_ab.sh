#!/bin/bash
# A/B of target-scan variants (AURORA_LIB selects a prebuilt library variant).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "full_parity_small or edge_shapes or all_rejected or status_word or llama_full_size or large_config or determinism" > gpurun_out/scan_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/scan_tests.log
for c in llama qwen3; do for v in "" B C D; do
  lib=paper_2602_06932_b200/libaurora${v:+_$v}.so
  AURORA_LIB=$PWD/$lib timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/sab_$c$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/sab_$c$v.json').read().strip().splitlines()[-1]); ph=d['phases_ms_per_step']; print('$c variant[$v]', d['ms_per_step'], 'scan', ph.get('target_scan'), d['clocks']['sm_mhz'])"
done; done

#!/bin/bash
# A/B of tree-attention variants (AURORA_LIB selects a prebuilt library variant).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export AURORA_TREE_FWD_TC=${AURORA_TREE_FWD_TC:-1}
for v in "" B C; do
  lib=paper_2602_06932_b200/libaurora${v:+_$v}.so
  AURORA_LIB=$PWD/$lib timeout 400 python bench.py --workload tree_attn --ta-config ${TA_CFG:-ta_tree} --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); print('variant[$v]', d['ms_per_step'], d['phases_ms_per_step'], d['clocks']['sm_mhz'])"
done
if [ -n "$1" ]; then AURORA_LIB=$PWD/paper_2602_06932_b200/libaurora_$1.so timeout 400 python -m pytest tests/test_gpu_tree_attn.py -q -x 2>&1 | tail -2; fi

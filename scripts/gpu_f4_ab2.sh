#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tree_attn.py -q -x > gpurun_out/f4_tests.log 2>&1; echo f4_tests_rc=$?; tail -2 gpurun_out/f4_tests.log
for c in ta_tree ta_llama; do
for v in "" B; do
  lib=paper_2602_06932_b200/libaurora${v:+_$v}.so
  AURORA_LIB=$PWD/$lib timeout 400 python bench.py --workload tree_attn --ta-config $c --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); print('$c variant[$v]', d['ms_per_step'], d['phases_ms_per_step'], d['clocks']['sm_mhz'])"
done; done

#!/bin/bash
# A/B: bulk L2 prefetch of the target-scan segments (option scan_prefetch).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -m paper_2602_06932_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "scan or verify or label or step" > gpurun_out/scan_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/scan_tests.log
for c in llama qwen3; do for v in 1 0; do
  AURORA_SCAN_PREFETCH=$v timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/sab_$c$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/sab_$c$v.json').read().strip().splitlines()[-1]); ph=d['phases_ms_per_step']; print('$c prefetch=$v', d['ms_per_step'], 'scan', ph.get('target_scan'), 'verify', ph.get('verify'), d['clocks']['sm_mhz'])"
done; done

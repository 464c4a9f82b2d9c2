#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build_failed; exit 1; }
for m in 0 4; do echo "== dbg_epi=$m"; AURORA_DBG_EPI=$m timeout 120 python scripts/store_microbench.py | grep umma; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "engine or full_parity or pair or accumulate" > gpurun_out/iter_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/iter_tests.log
for m in 0 4; do AURORA_DBG_EPI=$m timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench dbg=$m', d['ms_per_step'], d['phases_ms_per_step'])"; done

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for m in 0 8; do
  AURORA_DBG_EPI=$m timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > g.json 2>/dev/null
  python -c "import json; d=json.loads(open('g.json').read().strip().splitlines()[-1]); print('dbg=$m', d['ms_per_step'], d['phases_ms_per_step']['bwd_dw_gemm'], d['roofline']['frac'])"
done
cd scripts; for m in 0 8; do AURORA_DBG_EPI=$m MB_K=384 AURORA_DBG_NFAST=1 timeout 200 python store_microbench2.py | head -2; done

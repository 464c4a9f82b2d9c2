#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for env in "AURORA_BWD=classic" "AURORA_BWD=fused" "AURORA_SERIAL_BWD=0"; do
  env $env timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > g.json 2>/dev/null
  python -c "import json; d=json.loads(open('g.json').read().strip().splitlines()[-1]); print('$env', d['ms_per_step'], d['phases_ms_per_step'])"
  env $env timeout 300 python bench.py --config qwen3 --steps 10 --warmup 3 --no-cpu-baseline > g.json 2>/dev/null
  python -c "import json; d=json.loads(open('g.json').read().strip().splitlines()[-1]); print('  qwen3 $env', d['ms_per_step'])"
done

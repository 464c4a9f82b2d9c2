#!/bin/bash
# A/B: serial vs concurrent bwd (AURORA_SERIAL_BWD), llama + qwen3
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build_failed; tail -20 gpurun_out/build.log; exit 1; }
for cfg in llama qwen3; do
  for ser in 1 0; do
    AURORA_SERIAL_BWD=$ser timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${cfg}_${ser}.json 2>&1
    python - <<PY
import json
d = json.loads(open("gpurun_out/ab_${cfg}_${ser}.json").read().strip().splitlines()[-1])
print("${cfg} serial=${ser}", d["ms_per_step"], d["value"], d["phases_ms_per_step"], "e2e", d["e2e"]["ms_per_step"])
PY
  done
done

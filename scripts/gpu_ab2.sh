#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build_failed; exit 1; }
for cfg in llama qwen3 minimax; do
  for pair in 0 1; do
    AURORA_PAIR=$pair timeout 400 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab2_${cfg}_${pair}.json 2>&1
    python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/ab2_${cfg}_${pair}.json").read().strip().splitlines()[-1])
    print("${cfg} pair=${pair}", d["ms_per_step"], d["value"], d["tensor_frac_step"], d["phases_ms_per_step"])
except Exception as e:
    print("${cfg} pair=${pair} FAILED", open("gpurun_out/ab2_${cfg}_${pair}.json").read()[-600:])
PY
  done
done
AURORA_BWD=fused timeout 400 python bench.py --config qwen3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab2_q_fused.json 2>&1; tail -1 gpurun_out/ab2_q_fused.json | cut -c1-300

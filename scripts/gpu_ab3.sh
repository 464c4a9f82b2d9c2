#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build_failed; exit 1; }
for cfg in llama qwen3; do
  for ser in 0 1; do
    AURORA_SERIAL_BWD=$ser timeout 400 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab3_${cfg}_${ser}.json 2>&1
    python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/ab3_${cfg}_${ser}.json").read().strip().splitlines()[-1])
    r = d["roofline"]
    print("${cfg} serial=${ser}", d["ms_per_step"], d["value"], d["tensor_frac_step"], "roof", r["kernel"], r["bound"], r["frac"], d["phases_ms_per_step"])
except Exception as e:
    print("${cfg} serial=${ser} FAILED", open("gpurun_out/ab3_${cfg}_${ser}.json").read()[-600:])
PY
  done
done
AURORA_SERIAL_BWD=1 timeout 600 ncu --set full --clock-control none -k regex:k_umma_gemm -s 13 -c 1 -o gpurun_out/prof_fwd python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_fwd.log 2>&1; echo ncu_rc=$?

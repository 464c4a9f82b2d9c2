#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build_failed; tail -20 gpurun_out/build.log; exit 1; }
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -3 gpurun_out/smoke.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "not llama and not large" > gpurun_out/parity.log 2>&1; echo parity_rc=$?; tail -15 gpurun_out/parity.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "llama" > gpurun_out/parity_llama.log 2>&1; echo pl_rc=$?; tail -3 gpurun_out/parity_llama.log
for cfg in llama qwen3; do
  for mode in fused classic; do
    AURORA_BWD=$mode timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/f_${cfg}_${mode}.json 2>&1
    python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/f_${cfg}_${mode}.json").read().strip().splitlines()[-1])
    print("${cfg} ${mode}", d["ms_per_step"], d["value"], d["phases_ms_per_step"], "e2e", d["e2e"]["ms_per_step"])
except Exception as e:
    print("${cfg} ${mode} FAILED", open("gpurun_out/f_${cfg}_${mode}.json").read()[-800:])
PY
  done
done
timeout 200 python scripts/gemm_microbench.py mma > gpurun_out/micro_mma.jsonl 2>&1; cat gpurun_out/micro_mma.jsonl

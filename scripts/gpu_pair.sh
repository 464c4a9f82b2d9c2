#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build_failed; tail -20 gpurun_out/build.log; exit 1; }
timeout 200 python -m pytest tests/test_gpu_parity.py -q -x -k "cta_pair" > gpurun_out/pair.log 2>&1; echo pair_rc=$?; tail -15 gpurun_out/pair.log
timeout 400 python -m pytest tests/test_gpu_parity.py -q -k "not llama and not large and not cta_pair" > gpurun_out/parity.log 2>&1; echo parity_rc=$?; tail -8 gpurun_out/parity.log
for cfg in llama qwen3; do
  for pair in 0 1 2; do
    AURORA_PAIR=$pair timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/p_${cfg}_${pair}.json 2>&1
    python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/p_${cfg}_${pair}.json").read().strip().splitlines()[-1])
    print("${cfg} pair=${pair}", d["ms_per_step"], d["value"], d["phases_ms_per_step"])
except Exception as e:
    print("${cfg} pair=${pair} FAILED", open("gpurun_out/p_${cfg}_${pair}.json").read()[-600:])
PY
  done
done
timeout 200 python scripts/gemm_microbench.py mma > gpurun_out/micro_mma.jsonl 2>&1; AURORA_PAIR=2 timeout 200 python scripts/gemm_microbench.py mma >> gpurun_out/micro_mma.jsonl 2>&1; cat gpurun_out/micro_mma.jsonl

#!/bin/bash
# Iteration: build, targeted tests ($TESTS -k expr), bench llama (+qwen3), optional microbench.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build_failed; tail -20 gpurun_out/build.log; exit 1; }
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "$TESTS" > gpurun_out/iter_tests.log 2>&1; echo tests_rc=$?; tail -6 gpurun_out/iter_tests.log
fi
if [ -n "$MICRO" ]; then
  timeout 300 python $MICRO > gpurun_out/micro.jsonl 2>&1; echo micro_rc=$?; cat gpurun_out/micro.jsonl | tail -20
fi
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline ${BENCH_EXTRA} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python - <<'PY'
import json
for f in ["gpurun_out/bench.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], d["phases_ms_per_step"], d["roofline"]["frac"])
    except Exception as e:
        print(f, "ERR", e)
PY
tail -3 gpurun_out/bench.err
if [ -n "$QWEN" ]; then
  timeout 300 python bench.py --config qwen3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_qwen3.json 2>&1; echo bq_rc=$?
  tail -1 gpurun_out/bench_qwen3.json | cut -c1-1500
fi

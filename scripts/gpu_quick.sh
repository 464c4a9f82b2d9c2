#!/bin/bash
# Quick GPU iteration: build check, parity tests (fast subset), bench llama + qwen3.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build_failed; tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "not llama and not large" > gpurun_out/parity.log 2>&1; echo parity_rc=$?
tail -15 gpurun_out/parity.log
timeout 300 python bench.py --steps 20 --warmup 5 ${BENCH_EXTRA} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 300 python bench.py --config qwen3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_qwen3.json 2>&1; echo bq_rc=$?
tail -2 gpurun_out/bench_qwen3.json
if [ -n "$NCU_LAUNCHES" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo ncu1_rc=$?
fi
if [ -n "$NCU_FULL" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$NCU_FULL" -s ${NCU_SKIP:-0} -c ${NCU_COUNT:-3} -o gpurun_out/prof_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
fi
if [ -n "$MICRO" ]; then
  timeout 300 python scripts/gemm_microbench.py > gpurun_out/micro.jsonl 2>&1; echo micro_rc=$?
  cat gpurun_out/micro.jsonl
fi

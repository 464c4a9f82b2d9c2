#!/bin/bash
# Round-2 first GPU pass: build, smoke, every GPU test, default (qwen3) bench, llama bench,
# ncu launch list of the default bench.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02a; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log | cut -c1-300
timeout 1800 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1; echo gpu_tests_rc=$?; tail -3 $O/gpu_tests.log
run() { name=$1; shift; timeout 600 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | cut -c1-300; }
run qwen3
run llama --config llama --no-cpu-baseline
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_qwen3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --eager > $O/ncu_launches.log 2>&1; echo ncu_l_rc=$?

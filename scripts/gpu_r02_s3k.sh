#!/bin/bash
# C4 dH allreduce on the communicator's side stream (overlapped with dW): multi-rank parity.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/s3k; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -q -x -k "multirank or vocab or comm or dp" > $O/t_mr.log 2>&1; echo tmr_rc=$?; tail -1 $O/t_mr.log; grep -E "^(FAILED|E )" $O/t_mr.log | head -5
run() { name=$1; shift; timeout 240 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('phases_ms_per_step'))" 2>&1 | cut -c1-300; }
run comm1 --comm1 --no-cpu-baseline
run qwen3 --no-cpu-baseline

#!/bin/bash
# tcgen05 backward: lse / D loads hoisted before the ancestor walk; tests + timing.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/s3q; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_tree_attn.py -q -x > $O/t_attn.log 2>&1; echo tattn_rc=$?; tail -1 $O/t_attn.log; grep -E "^(FAILED|E )" $O/t_attn.log | head -5
run() { name=$1; shift; timeout 240 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('phases_ms_per_step'))" 2>&1 | cut -c1-300; }
run t1 --workload tree_attn --ta-config ta_tree --no-cpu-baseline
run t2 --workload tree_attn --ta-config ta_tree --no-cpu-baseline
run l1 --workload tree_attn --ta-config ta_llama --no-cpu-baseline

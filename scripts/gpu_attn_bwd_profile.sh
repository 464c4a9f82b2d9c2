#!/bin/bash
# tcgen05 backward with 8 compute warps: tests, timings, ncu.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/s3g; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_tree_attn.py -q -x > $O/t_attn.log 2>&1; echo tattn_rc=$?; tail -1 $O/t_attn.log; grep -E "^(FAILED|E )" $O/t_attn.log | head -5
run() { name=$1; shift; timeout 240 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('phases_ms_per_step'), d['roofline']['frac'])" 2>&1 | cut -c1-300; }
run ta_tree --workload tree_attn --ta-config ta_tree --no-cpu-baseline
run ta_llama --workload tree_attn --ta-config ta_llama --no-cpu-baseline
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_ta_bwd_tc" -c 1 -o $O/prof_btc -f python bench.py --workload tree_attn --ta-config ta_tree --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_btc.log 2>&1; echo ncu_btc_rc=$?

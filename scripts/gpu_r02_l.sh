#!/bin/bash
# tcgen05 one-pass tree attention with P in TMEM (tree_fwd_tc 4 / 5): parity under a short
# timeout, then benches against the mma.sync forward and the smem-P variant.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02l; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 240 python -m pytest tests/test_gpu_tree_attn.py -q -x -k "tc4 or tc5" > $O/t_pt.log 2>&1; echo pt_rc=$?; tail -2 $O/t_pt.log; grep -E "^E " $O/t_pt.log | head -8
run() { name=$1; shift; timeout 300 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | cut -c1-120; tail -2 $O/b_$name.err; }
for f in 0 2 4 5; do
  AURORA_TREE_FWD_TC=$f run tree_f$f --workload tree_attn --ta-config ta_tree --no-cpu-baseline
  AURORA_TREE_FWD_TC=$f run llama_f$f --workload tree_attn --ta-config ta_llama --no-cpu-baseline
done
AURORA_TREE_FWD_TC=4 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_ta_fwd_tc2" -c 1 -o $O/prof_tc4 -f python bench.py --workload tree_attn --ta-config ta_tree --steps 1 --warmup 1 --no-cpu-baseline --eager > $O/ncu.log 2>&1; echo ncu_rc=$?

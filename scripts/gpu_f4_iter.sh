#!/bin/bash
# F4 iteration: parity, bench lines, ncu of the tree-attention kernels.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -m paper_2602_06932_b200.build > /dev/null
timeout 600 python -m pytest tests/test_gpu_tree_attn.py -q -x > gpurun_out/f4_tests.log 2>&1; echo f4_tests_rc=$?; tail -3 gpurun_out/f4_tests.log
for c in ta_tree ta_llama; do
  timeout 400 python bench.py --workload tree_attn --ta-config $c --no-cpu-baseline > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; echo ${c}_rc=$?
  python -c "
import json; d=json.loads(open('gpurun_out/b_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['value'], d['phases_ms_per_step'], [(p['kernel'], p['achieved_gbs'], p['achieved_tflops']) for p in d['roofline']['phases']], d['clocks']['sm_mhz'])"
done
if [ "$1" = "prof" ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ta_ -c 4 -o gpurun_out/prof_ta_tree -f python bench.py --workload tree_attn --ta-config ta_tree --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_ta.log 2>&1; echo ncu_rc=$?
fi

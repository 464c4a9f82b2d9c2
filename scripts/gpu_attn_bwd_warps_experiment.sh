#!/bin/bash
# tcgen05 backward with 16 compute warps (4 per TMEM lane quadrant): parity + timing vs 8 warps.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/s3o; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
python -c "from paper_2602_06932_b200.build import *; import subprocess,os; srcs=[os.path.join(CSRC,s) for s in SOURCES]; subprocess.run([NVCC,*FLAGS,'-DTA_BWD_CW=8','-I',os.path.join(ROOT,'include'),'-o','/tmp/libaurora_cw8.so',*srcs,'-ldl'],check=True)" > $O/build2.log 2>&1; echo build2_rc=$?
timeout 600 python -m pytest tests/test_gpu_tree_attn.py -q -x > $O/t_attn.log 2>&1; echo tattn_rc=$?; tail -1 $O/t_attn.log; grep -E "^(FAILED|E )" $O/t_attn.log | head -5
run() { name=$1; shift; timeout 240 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('phases_ms_per_step'))" 2>&1 | cut -c1-300; }
run cw16 --workload tree_attn --ta-config ta_tree --no-cpu-baseline
AURORA_LIB=/tmp/libaurora_cw8.so run cw8 --workload tree_attn --ta-config ta_tree --no-cpu-baseline
run cw16b --workload tree_attn --ta-config ta_tree --no-cpu-baseline
run cw16_llama --workload tree_attn --ta-config ta_llama --no-cpu-baseline
AURORA_LIB=/tmp/libaurora_cw8.so run cw8_llama --workload tree_attn --ta-config ta_llama --no-cpu-baseline

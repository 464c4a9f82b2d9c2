#!/bin/bash
# Experiment: time of the tcgen05 backward with the dV^T / dK^T MMAs cut to 1 K step (wrong
# results, timing only) -> upper bound of what cheaper gradient MMAs can buy.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/s3n; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
python -c "from paper_2602_06932_b200.build import *; import subprocess,os; srcs=[os.path.join(CSRC,s) for s in SOURCES]; subprocess.run([NVCC,*FLAGS,'-DTA_BWD_NO_KV_STORE','-I',os.path.join(ROOT,'include'),'-o','/tmp/libaurora_nostore.so',*srcs,'-ldl'],check=True)" > $O/build2.log 2>&1; echo build2_rc=$?
run() { name=$1; shift; timeout 240 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('phases_ms_per_step'))" 2>&1 | cut -c1-300; }
run base --workload tree_attn --ta-config ta_tree --no-cpu-baseline
AURORA_LIB=/tmp/libaurora_nostore.so run nostore --workload tree_attn --ta-config ta_tree --no-cpu-baseline

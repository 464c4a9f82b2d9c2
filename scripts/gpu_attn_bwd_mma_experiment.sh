#!/bin/bash
# Experiments (timing only, wrong results): tcgen05 backward with the dP MMAs cut to 1 K step, and
# with both dP and dV^T / dK^T cut -> how much of the time is shared-memory operand traffic.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/s3p; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
bld() { python -c "from paper_2602_06932_b200.build import *; import subprocess,os,sys; srcs=[os.path.join(CSRC,s) for s in SOURCES]; subprocess.run([NVCC,*FLAGS,*sys.argv[2:],'-I',os.path.join(ROOT,'include'),'-o',sys.argv[1],*srcs,'-ldl'],check=True)" "$@" >> $O/build2.log 2>&1; echo build_rc=$?; }
bld /tmp/lib_dp1.so -DTA_BWD_DP_KSTEPS=1
bld /tmp/lib_dp1kv1.so -DTA_BWD_DP_KSTEPS=1 -DTA_BWD_KV_KSTEPS=1
run() { name=$1; shift; timeout 240 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('phases_ms_per_step'))" 2>&1 | cut -c1-300; }
run base --workload tree_attn --ta-config ta_tree --no-cpu-baseline
AURORA_LIB=/tmp/lib_dp1.so run dp1 --workload tree_attn --ta-config ta_tree --no-cpu-baseline
AURORA_LIB=/tmp/lib_dp1kv1.so run dp1kv1 --workload tree_attn --ta-config ta_tree --no-cpu-baseline

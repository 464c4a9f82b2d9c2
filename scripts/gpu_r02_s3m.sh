#!/bin/bash
# F3 fused AdamW: state-entry shapes (dw_adamw_qe 0 / 1 / 2).
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/s3m; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
run() { name=$1; shift; timeout 240 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('phases_ms_per_step'))" 2>&1 | cut -c1-300; }
for q in 1 2 0 1 2; do AURORA_DW_ADAMW_QE=$q run f3_q$q --config llama --optimizer fused --no-cpu-baseline; done

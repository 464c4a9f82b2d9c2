#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/dl
python -m paper_2602_06932_b200.build > /dev/null
for c in ta_llama ta_tree; do
  timeout 600 python bench.py --workload draft_layer --ta-config $c --steps 10 > gpurun_out/dl/b_dl_$c.json 2> gpurun_out/dl/b_dl_$c.err; echo ${c}_rc=$?; tail -1 gpurun_out/dl/b_dl_$c.json | cut -c1-1500; tail -3 gpurun_out/dl/b_dl_$c.err
done

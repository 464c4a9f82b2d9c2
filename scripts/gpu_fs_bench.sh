#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/fs
python -m paper_2602_06932_b200.build > /dev/null
for c in llama tree; do
  timeout 900 python bench.py --workload full_step --config $c --steps 10 > gpurun_out/fs/b_fs_$c.json 2> gpurun_out/fs/b_fs_$c.err; echo ${c}_rc=$?; tail -1 gpurun_out/fs/b_fs_$c.json | cut -c1-1200; tail -3 gpurun_out/fs/b_fs_$c.err
done

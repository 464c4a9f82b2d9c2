#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/fs
python -m paper_2602_06932_b200.build > /dev/null
for opt in "" "--optimizer"; do
  timeout 900 python bench.py --workload full_step --config llama --steps 10 $opt > gpurun_out/fs/b_fs_llama$opt.json 2> gpurun_out/fs/b_fs_llama$opt.err; echo llama${opt}_rc=$?; tail -1 gpurun_out/fs/b_fs_llama$opt.json | cut -c1-600; tail -3 gpurun_out/fs/b_fs_llama$opt.err
done

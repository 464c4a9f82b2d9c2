#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build_failed; exit 1; }
timeout 300 compute-sanitizer --tool memcheck python scripts/f2_repro.py tiny 2>&1 | head -60
timeout 300 python -m pytest tests/test_gpu_optim.py -q -x 2>&1 | tail -15

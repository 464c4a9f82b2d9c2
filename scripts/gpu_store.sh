#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build_failed; exit 1; }
cd scripts
for nf in 0 1; do AURORA_DBG_NFAST=$nf timeout 200 python store_microbench2.py; done
MB_K=384 AURORA_DBG_NFAST=1 timeout 200 python store_microbench2.py

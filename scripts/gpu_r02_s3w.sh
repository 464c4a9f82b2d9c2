#!/bin/bash
# Tree attention: prefix edge lengths (empty / exactly full tiles) for every default kernel.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/s3w; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_tree_attn.py tests/test_gpu_fullsize.py -q -k "edge or top16" > $O/t.log 2>&1; echo t_rc=$?; tail -3 $O/t.log; grep -E "^(FAILED|E )" $O/t.log | head -8

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build_failed; tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_optim.py -q -x > gpurun_out/t_optim.log 2>&1; echo optim_rc=$?; tail -25 gpurun_out/t_optim.log
pr() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']; print(sys.argv[2], d['ms_per_step'], d['value'], d['phases_ms_per_step'], r['kernel'], r['achieved'], r['frac'])" $1 "$2"; }
for o in fused unfused; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --optimizer $o > gpurun_out/g.json 2> gpurun_out/g.err; echo "rc=$?"; pr gpurun_out/g.json "opt=$o"; tail -2 gpurun_out/g.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dw_resident or full_parity or multi_chunk" > gpurun_out/t.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t.log

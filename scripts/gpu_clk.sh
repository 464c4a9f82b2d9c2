#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build_failed; exit 1; }
timeout 400 python bench.py > gpurun_out/b_default.json 2> gpurun_out/b_default.err; echo rc=$?
python -c "import json; d=json.loads(open('gpurun_out/b_default.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['clocks'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'])"
tail -3 gpurun_out/b_default.err
timeout 400 python bench.py --eager --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_eager.json 2>&1; echo rc=$?; python -c "import json; d=json.loads(open('gpurun_out/b_eager.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks'])"
timeout 400 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/b_ref.json 2>&1; echo ref_rc=$?; tail -1 gpurun_out/b_ref.json | cut -c1-400

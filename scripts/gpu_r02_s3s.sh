#!/bin/bash
# k_dz_rescale without per-element index arithmetic: parity + timings.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/s3s; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build_failed; tail -20 $O/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "not scan" > $O/t_par.log 2>&1; echo tpar_rc=$?; tail -1 $O/t_par.log; grep -E "^(FAILED|E )" $O/t_par.log | head -5
run() { name=$1; shift; timeout 600 python bench.py "$@" > $O/b_$name.json 2> $O/b_$name.err; echo ${name}_rc=$?; tail -1 $O/b_$name.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k:v for k,v in d.get('phases_ms_per_step').items() if v>0.03})" 2>&1 | cut -c1-300; }
run qwen3 --no-cpu-baseline
run llama --config llama --no-cpu-baseline
run tree --config tree --no-cpu-baseline

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build_failed; exit 1; }
pr() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d['ms_per_step'], d['value'], d['config'].get('launch'), d['gpu_launches'], d['phases_ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['traffic'])" $1 "$2"; }
for extra in "" "--eager" "--optimizer" "--target-topk 1024"; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline $extra > gpurun_out/g.json 2> gpurun_out/g.err; echo "rc=$? [$extra]"; pr gpurun_out/g.json "[$extra]"; tail -2 gpurun_out/g.err
done
for sc in 1 4 8; do
  AURORA_SCAN_CTAS=$sc timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g.json 2> gpurun_out/g.err; pr gpurun_out/g.json "scan_ctas=$sc"
done
for tn in 256 224; do
  AURORA_TILE_N=$tn timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g.json 2> gpurun_out/g.err; pr gpurun_out/g.json "tile_n=$tn"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "full_parity or topk_ingest_parity or edge or status or llama" > gpurun_out/t.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t.log

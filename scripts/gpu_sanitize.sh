#!/bin/bash
# compute-sanitizer on the tiny smoke path (all kernels), default + pair + fused modes.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  for env in "" "AURORA_PAIR=2" "AURORA_BWD=fused"; do
    env $env timeout 600 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_${tool}_${env%%=*}.log 2>&1
    echo "$tool [$env] rc=$? :: $(grep -E 'ERROR SUMMARY|smoke ok' gpurun_out/san_${tool}_${env%%=*}.log | tr '\n' ' ' | cut -c1-200)"
  done
done

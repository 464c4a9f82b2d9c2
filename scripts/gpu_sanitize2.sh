#!/bin/bash
# compute-sanitizer over the newer paths (F1 long supports, F2 objectives, F3 AdamW).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/san_variants.py > gpurun_out/san2_${tool}.log 2>&1
  echo "$tool rc=$? :: $(grep -E 'ERROR SUMMARY|variants ok' gpurun_out/san2_${tool}.log | tr '\n' ' ' | cut -c1-200)"
done

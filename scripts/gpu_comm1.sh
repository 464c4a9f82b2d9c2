#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
pr() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d['ms_per_step'], d['value'], d['config']['parallelism'], d['config']['launch'], d['roofline']['frac'], (d.get('e2e') or {}).get('value'))" $1 "$2"; }
for extra in "" "--comm1" "--comm1 --accept-loss rkl --ntp-beta 0.5 --k-discard 0" "--comm1 --optimizer"; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $extra > g.json 2> g.err; echo "rc=$? [$extra]"; pr g.json "[$extra]"; tail -2 g.err
done

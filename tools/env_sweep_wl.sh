#!/bin/bash
# solve time of workload $1 under environment-knob variants: bash tools/env_sweep_wl.sh c2w "" "PMG_MID_NODES=0"
wl=$1; shift
for v in "$@"; do
  env $v python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline > /tmp/es.json 2>/dev/null
  echo "[$wl $v] $(python -c "import json; d=json.loads(open('/tmp/es.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), 'ms/solve')")"
done

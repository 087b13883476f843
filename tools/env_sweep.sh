#!/bin/bash
# c1 solve time under environment-knob variants:
#   bash tools/env_sweep.sh "" "PMG_MID_NODES=0" "PMG_MID_CLUSTER=8" ...
for v in "$@"; do
  env $v python bench.py --steps 10 --no-cpu-baseline > /tmp/es.json 2>/dev/null
  echo "[$v] $(python -c "import json; d=json.loads(open('/tmp/es.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), 'ms/solve')")"
done

#!/bin/bash
# c3 ms/solve and radial roofline under launch-shape overrides
run() { echo -n "$1: "; env $2 python bench.py --workload c3 --steps 3 > /tmp/s.json 2>/dev/null; python -c "import json; d=json.loads(open('/tmp/s.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],2), d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['ms_per_launch'])"; }
run default ""
run maxt128 "PMG_LINE_MAXT=128"
run maxt64 "PMG_LINE_MAXT=64"
run maxt512 "PMG_LINE_MAXT=512"

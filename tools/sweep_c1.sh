#!/bin/bash
# c1 ms/solve under launch-shape environment overrides
run() { echo -n "$1: "; env $2 python bench.py --steps 10 > /tmp/s.json 2>/dev/null; python -c "import json; d=json.loads(open('/tmp/s.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), d['roofline']['frac'])"; }
run default ""
run maxt512 "PMG_LINE_MAXT=512"
run maxt128 "PMG_LINE_MAXT=128"
run maxt64 "PMG_LINE_MAXT=64"

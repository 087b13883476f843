#!/bin/bash
# A/B of two library builds on the default bench: bash tools/ab_lib.sh libA.so libB.so
for i in 1 2 3; do
for L in "$@"; do
PMG_LIB=paper_2507_03812_b200/lib/$L python bench.py --steps 20 > /tmp/s.json 2>/dev/null
echo "$L $(python -c "import json; d=json.loads(open('/tmp/s.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), d['roofline']['frac'])")"
done; done

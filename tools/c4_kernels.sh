#!/bin/bash
# per-kernel ms and roofline fraction of the config-4 microbench
python bench.py --workload c4 --reps ${1:-20} > /tmp/c4.json 2>/dev/null
python - <<'PY'
import json
d = json.loads(open("/tmp/c4.json").read().strip().splitlines()[-1])
for k, v in d["kernels"].items():
    print(f"{k:9s} {v['ms_per_launch']:.4f} ms  {v['achieved']:.0f} GB/s  frac {v['frac']:.3f}")
PY

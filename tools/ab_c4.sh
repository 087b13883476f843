#!/bin/bash
# A/B of library builds on the config-4 kernel microbench:
#   bash tools/ab_c4.sh libA.so libB.so ...   (names under paper_2507_03812_b200/lib/)
for L in "$@"; do
  PMG_LIB=paper_2507_03812_b200/lib/$L python bench.py --workload c4 --reps 20 > /tmp/c4ab.json 2>/dev/null
  python - "$L" <<'PY'
import json, sys
d = json.loads(open("/tmp/c4ab.json").read().strip().splitlines()[-1])
print(sys.argv[1], "  ".join(f"{k} {v['ms_per_launch']:.4f} ms ({v['frac']:.3f})" for k, v in d["kernels"].items()))
PY
done

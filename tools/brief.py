"""One-screen summary of a gpurun_out/<dir>: pytest tail + bench lines."""
import glob
import json
import os
import sys

d = sys.argv[1]
p = os.path.join(d, "pytest.txt")
if os.path.exists(p):
    print("".join(open(p).readlines()[-14:]))
for f in sorted(glob.glob(os.path.join(d, "bench_*.json"))):
    try:
        j = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(os.path.basename(f), "no json:", open(f.replace(".json", ".err")).read()[-600:])
        continue
    bd = j.get("breakdown_one_solve", {})
    ks = j.get("kernels_finest_level", {})
    print(f"{os.path.basename(f)}: {j.get('ms_per_step', 0):.2f} ms/step value {j.get('value', 0):.3e} "
          f"e2e {j.get('e2e', {}).get('value', 0):.3e} its {j.get('run_info', {}).get('iterations_first_sections')}")
    print("   breakdown ms: " + " ".join(f"{k}={v['ms']:.2f}" for k, v in bd.items()))
    print("   finest frac: " + " ".join(f"{k}={v.get('frac')}({v.get('ms_per_launch')}ms)" for k, v in ks.items()))

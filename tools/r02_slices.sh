#!/bin/bash
# per-rank workload of the sharded config-3 batch on one GPU: the slice rank 0 of an N-GPU job owns
out=${1:-gpurun_out/r02slices}
mkdir -p $out
for n in 1 2 4 8; do
  python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --rank-slice $n > $out/slice_$n.json 2> $out/slice_$n.err
done
python - <<PY
import json
t = {}
for n in (1, 2, 4, 8):
    j = json.loads(open("$out/slice_%d.json" % n).read().strip().splitlines()[-1])
    t[n] = (j["ms_per_step"], j["value"], j["e2e"]["value"], j["run_info"]["sections_per_rank"])
print("| N (GPUs emulated) | sections per rank | ms per solve of the rank's slice | rank DOF*cycles/s | projected N-GPU throughput (N x rank) | projected speed-up vs N=1 |")
print("|---|---|---|---|---|---|")
for n in (1, 2, 4, 8):
    ms, v, e, b = t[n]
    print(f"| {n} | {b} | {ms:.2f} | {v:.3e} | {n * v:.3e} | {t[1][0] / ms:.2f}x |")
PY

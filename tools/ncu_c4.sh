#!/bin/bash
# ncu --set full captures of the config-4 (8193x8192) finest-level kernels.
# usage (on the GPU box): bash tools/ncu_c4.sh <outdir>
out=${1:-gpurun_out/ncu}
mkdir -p $out
for k in k_apply_tma k_circle_cl k_radial_cl; do
  ncu --set full --clock-control none --import-source on -k regex:"^${k}" -c 2 \
      -o $out/c4_$k -f python bench.py --workload c4 --reps 1 > $out/c4_$k.log 2>&1
  python tools/ncu_summary.py $out/c4_$k.ncu-rep > $out/c4_$k.md 2>&1
done

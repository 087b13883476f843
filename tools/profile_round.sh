#!/bin/bash
# Round evidence on one B200: bench lines, reference arm, ncu launch lists and
# --set full captures of the finest-level kernels.  usage: bash tools/profile_round.sh <out>
out=${1:-gpurun_out/r01c}
mkdir -p $out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > $out/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)|Thread|Core" > $out/host.txt
python bench.py > $out/bench_c1.json 2> $out/bench_c1.err
python bench.py --impl reference --steps 5 --warmup 1 > $out/ref_c1.json 2> $out/ref_c1.err
for w in c0 c2v c2w c3; do
  python bench.py --workload $w --steps 5 --warmup 3 > $out/bench_$w.json 2> $out/bench_$w.err
done
python bench.py --workload c4 --reps 50 > $out/bench_c4.json 2> $out/bench_c4.err
# launch list of the default bench command (cold-cache, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c1.csv \
    python bench.py --steps 3 --warmup 3 > $out/launches_c1.log 2>&1
python tools/summarize_launches.py $out/launches_c1.csv > $out/launches_c1.md
# per-level launch list of one warm solve (cache control none)
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file $out/levels_c1.csv python tools/solve_once.py 1 V 1 > /dev/null 2>&1
python tools/ncu_levels.py $out/levels_c1.csv > $out/levels_c1.md
# --set full of the finest-level kernels at 1025x1024 (first launches = level 0)
for k in k_apply_tiled k_smooth_fused; do
  ncu --set full --clock-control none --import-source on -k regex:"^${k}$" -c 2 \
      -o $out/c1_$k -f python tools/solve_once.py 1 V 1 > $out/c1_$k.log 2>&1
  python tools/ncu_summary.py $out/c1_$k.ncu-rep > $out/c1_$k.md 2>&1
done
bash tools/ncu_c4.sh $out
# keep what travels back under gpurun's 64 MiB: summaries, logs, and the c1 reports
du -sh $out/* | sort -h | tail -8
rm -f $out/launches_c1.csv $out/levels_c1.csv
for f in $out/*.ncu-rep; do
  [ $(stat -c %s $f) -gt 12000000 ] && rm -f $f
done
du -sh $out

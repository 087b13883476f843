out=${1:-gpurun_out/r01e}
mkdir -p $out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > $out/gpu.txt
python bench.py > $out/bench_c1.json 2> $out/bench_c1.err
python bench.py --impl reference --steps 5 --warmup 1 > $out/ref_c1.json 2> $out/ref_c1.err
for w in c0 c2v c2w c3; do
  python bench.py --workload $w --steps 5 --warmup 3 > $out/bench_$w.json 2> $out/bench_$w.err
done
python bench.py --workload c4 --reps 50 > $out/bench_c4.json 2> $out/bench_c4.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c1.csv \
    python bench.py --steps 3 --warmup 3 > $out/launches_c1.log 2>&1
python tools/summarize_launches.py $out/launches_c1.csv > $out/launches_c1.md
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file $out/levels_c1.csv python tools/solve_once.py 1 V 1 > /dev/null 2>&1
python tools/ncu_levels.py $out/levels_c1.csv > $out/levels_c1.md
ncu --set full --clock-control none --import-source on -k regex:"^k_smooth_fused" -c 1 \
    -o $out/c1_k_smooth_fused -f python tools/solve_once.py 1 V 1 > $out/c1_k_smooth_fused.log 2>&1
python tools/summarize_launches.py $out/launches_c1.csv > /dev/null
python tools/ncu_summary.py $out/c1_k_smooth_fused.ncu-rep > $out/c1_k_smooth_fused.md 2>&1
rm -f $out/launches_c1.csv $out/levels_c1.csv

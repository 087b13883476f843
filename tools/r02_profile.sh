#!/bin/bash
# Round-2 evidence on one B200: bench lines of every workload (benched = reference-order mode,
# plus the opt-in fast mode), the reference arm, the ncu launch list of the default bench
# command, and --set full captures of the config-3 finest-level kernels.
# usage: bash tools/r02_profile.sh <out>
out=${1:-gpurun_out/r02p}
mkdir -p $out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > $out/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)|Thread|Core" > $out/host.txt
timeout 1800 python -m pytest tests -q -m gpu --durations=8 > $out/pytest.txt 2>&1
echo "pytest rc=$?" >> $out/pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1
python bench.py > $out/bench_c3.json 2> $out/bench_c3.err
python bench.py --impl reference --steps 2 --warmup 1 > $out/ref_c3.json 2> $out/ref_c3.err
for w in c1 c2v c2w c0; do
  python bench.py --workload $w --steps 5 --warmup 3 > $out/bench_$w.json 2> $out/bench_$w.err
done
for w in c3 c1 c2v c2w c0; do
  python bench.py --workload $w --steps 5 --warmup 3 --fast --no-cpu-baseline --no-extras > $out/bench_${w}_fast.json 2> $out/bench_${w}_fast.err
done
python bench.py --workload c4 --reps 50 > $out/bench_c4.json 2> $out/bench_c4.err
python bench.py --workload c4 --reps 50 --fast > $out/bench_c4_fast.json 2> $out/bench_c4_fast.err
python bench.py --workload give --reps 20 > $out/bench_give.json 2> $out/bench_give.err
python tools/brief.py $out > $out/brief.txt 2>&1
# launch list of the default bench command (cold-cache, serialised: shares, not absolutes)
# (PMG_LOOP_GRAPH=0: kernel nodes of a conditional graph are invisible to ncu, so the solve loop
# runs as per-cycle graph launches here -- the same kernels)
PMG_LOOP_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c3.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extras > $out/launches_c3.log 2>&1
python tools/summarize_launches.py $out/launches_c3.csv > $out/launches_c3.md
# --set full of the config-3 finest-level kernels (third launch = warm)
ncu --set full --clock-control none --import-source on -k regex:"k_radial_warp" -s 2 -c 1 \
    -o $out/c3_radial_warp -f python tools/sweep_once.py 3 0 1 0 > $out/c3_radial_warp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_circle_warp" -s 2 -c 1 \
    -o $out/c3_circle_warp -f python tools/sweep_once.py 3 0 0 1 > $out/c3_circle_warp.log 2>&1
PMG_LOOP_GRAPH=0 ncu --set full --clock-control none --import-source on -k regex:"k_apply_tma" -s 2 -c 1 \
    -o $out/c3_apply_tma -f python tools/solve_once.py 3 V 1 > $out/c3_apply_tma.log 2>&1
for k in c3_radial_warp c3_circle_warp c3_apply_tma; do
  python tools/ncu_summary.py $out/$k.ncu-rep > $out/$k.md 2>&1
done
rm -f $out/launches_c3.csv
for f in $out/*.ncu-rep; do
  [ $(stat -c %s $f) -gt 20000000 ] && rm -f $f
done
tail -3 $out/pytest.txt; cat $out/smoke.txt | tail -3; cat $out/brief.txt
cat $out/c3_*.md
du -sh $out

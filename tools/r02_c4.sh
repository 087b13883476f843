#!/bin/bash
out=${1:-gpurun_out/r02q}
mkdir -p $out
timeout 1500 python -m pytest tests -q -m gpu -x --durations=8 > $out/pytest.txt 2>&1
echo "pytest rc=$?" >> $out/pytest.txt
tail -14 $out/pytest.txt
python bench.py --workload c4 --reps 50 > $out/bench_c4.json 2> $out/bench_c4.err
python bench.py --workload c4 --reps 50 --fast > $out/bench_c4_fast.json 2> $out/bench_c4_fast.err
for f in $out/bench_c4.json $out/bench_c4_fast.json; do python -c "
import json,sys; j=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', {k:(v['ms_per_launch'],v['frac']) for k,v in j['kernels'].items()})"; done
# launch list of the default bench command; the WHILE-graph's kernel nodes are invisible to ncu
# (conditional graphs are not profilable), so the solve loop runs as per-cycle graph launches here
PMG_LOOP_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c3.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $out/launches_c3.log 2>&1
python tools/summarize_launches.py $out/launches_c3.csv > $out/launches_c3.md
rm -f $out/launches_c3.csv
PMG_LOOP_GRAPH=0 ncu --set full --clock-control none --import-source on -k regex:"k_apply_tma" -s 2 -c 1 \
    -o $out/c3_apply_tma -f python tools/solve_once.py 3 V 1 > $out/c3_apply_tma.log 2>&1
python tools/ncu_summary.py $out/c3_apply_tma.ncu-rep > $out/c3_apply_tma.md 2>&1
cat $out/c3_apply_tma.md; head -12 $out/launches_c3.md

#!/bin/bash
# ncu --set full captures of the config-3 finest-level sweeps (exact mode): radial warp kernel, circle kernel
out=${1:-gpurun_out/r02b}
mkdir -p $out
timeout 600 python -m pytest tests/test_binding.py tests/test_gpu_determinism.py tests/test_gpu_configs.py -q -m gpu -x > $out/pytest.txt 2>&1
echo "pytest rc=$?" >> $out/pytest.txt
tail -5 $out/pytest.txt
for w in c3 c1 c0; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_$w.json 2> $out/bench_$w.err
done
PMG_LOOP_GRAPH=0 timeout 600 python bench.py --workload c1 --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_c1_noloop.json 2> $out/bench_c1_noloop.err
python tools/brief.py $out
# third launch of each kernel = warm
ncu --set full --clock-control none --import-source on -k regex:"k_radial_warp" -s 2 -c 1 \
    -o $out/c3_radial_warp -f python tools/sweep_once.py 3 0 1 0 > $out/c3_radial_warp.log 2>&1
python tools/ncu_summary.py $out/c3_radial_warp.ncu-rep > $out/c3_radial_warp.md 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_circle" -s 2 -c 1 \
    -o $out/c3_circle -f python tools/sweep_once.py 3 0 0 1 > $out/c3_circle.log 2>&1
python tools/ncu_summary.py $out/c3_circle.ncu-rep > $out/c3_circle.md 2>&1
cat $out/c3_radial_warp.md $out/c3_circle.md
ls -la $out

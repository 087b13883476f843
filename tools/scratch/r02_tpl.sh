#!/bin/bash
# thread-per-line radial sweep: parity tests, c3 bench (exact + fast), ncu capture
out=${1:-gpurun_out/r02c}
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_configs.py::test_config3_all_sections tests/test_gpu_determinism.py -q -m gpu -x > $out/pytest.txt 2>&1
echo "pytest rc=$?" >> $out/pytest.txt
tail -5 $out/pytest.txt
timeout 600 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_c3.json 2> $out/bench_c3.err
for g in $TPL_GS; do
PMG_TPL_G=$g timeout 600 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_c3_g$g.json 2> $out/bench_c3_g$g.err
done
python tools/brief.py $out
ncu --set full --clock-control none --import-source on -k regex:"k_radial_tpl" -s 2 -c 1 \
    -o $out/c3_radial_tpl -f python tools/sweep_once.py 3 0 1 0 > $out/c3_radial_tpl.log 2>&1
python tools/ncu_summary.py $out/c3_radial_tpl.ncu-rep > $out/c3_radial_tpl.md 2>&1
cat $out/c3_radial_tpl.md

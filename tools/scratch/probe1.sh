set -x
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv
./tools/scratch/dplat
for ro in "" "--reference-order"; do
  timeout 300 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline $ro > gpurun_out/p1_c3$ro.json 2>&1
  timeout 300 python bench.py --workload c1 --steps 5 --warmup 3 --no-cpu-baseline $ro > gpurun_out/p1_c1$ro.json 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/p1_pytest.log 2>&1
tail -25 gpurun_out/p1_pytest.log

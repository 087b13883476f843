#!/bin/bash
# exact-parallel line solves: GPU tests + reference-order benches
out=${1:-gpurun_out/r02b}
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> $out/pytest_gpu.txt
for w in ${WLS:-c1 c3 c2v c0 c2w}; do
  timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --reference-order \
      > $out/bench_${w}_ro.json 2> $out/bench_${w}_ro.err
done

#!/bin/bash
# exact-parallel line solves: wave traces + reference-order benches (+ optional tests)
out=${1:-gpurun_out/r02d}
mkdir -p $out
python tools/ktrace_ex.py 1 3 > $out/kt_c1.txt 2>&1
python tools/ktrace_ex.py 3 1 > $out/kt_c3.txt 2>&1
python tools/ktrace_ex.py 2 1 > $out/kt_c2.txt 2>&1
for w in ${WLS:-c1 c3 c2v}; do
  timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --reference-order \
      > $out/bench_${w}_ro.json 2> $out/bench_${w}_ro.err
done
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.txt; fi

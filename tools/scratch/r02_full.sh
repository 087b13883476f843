#!/bin/bash
# round-2 evidence: full GPU test suite, then bench lines (exact and fast mode) for every workload
out=${1:-gpurun_out/r02a}
mkdir -p $out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > $out/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)|Thread|Core" > $out/host.txt
timeout 3000 python -m pytest tests -q -m gpu --durations=15 > $out/pytest.txt 2>&1
echo "pytest rc=$?" >> $out/pytest.txt
for w in c3 c1 c2v c2w c0; do
  for m in "" "--fast"; do
    tag=$w${m:+_fast}
    timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline $m \
      > $out/bench_$tag.json 2> $out/bench_$tag.err
  done
done
timeout 900 python bench.py --workload c4 --reps 50 > $out/bench_c4.json 2> $out/bench_c4.err
timeout 900 python bench.py --workload c4 --reps 50 --fast > $out/bench_c4_fast.json 2> $out/bench_c4_fast.err
python tools/brief.py $out > $out/brief.txt 2>&1
cat $out/brief.txt

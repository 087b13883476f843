#!/bin/bash
# round-2 first GPU probe: tests + both line-solve modes on every config
out=${1:-gpurun_out/r02a}
mkdir -p $out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > $out/gpu.txt
lscpu | head -20 > $out/host.txt
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> $out/pytest_gpu.txt
for w in c3 c1 c2v c2w c0; do
  for ro in "" "--reference-order"; do
    tag=$w${ro:+_ro}
    timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline $ro \
      > $out/bench_$tag.json 2> $out/bench_$tag.err
  done
done

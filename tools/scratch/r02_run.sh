#!/bin/bash
# round-2 iteration run: selected GPU tests, then c3 bench lines in both modes
# usage: tools/r02_run.sh OUT "pytest args" "workloads"
out=${1:-gpurun_out/r02x}
tests=${2:-"tests/test_gpu_configs.py"}
wls=${3:-"c3"}
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv > $out/gpu.txt
if [ "$tests" != "none" ]; then
  timeout 1500 python -m pytest $tests -x -q -m gpu --durations=10 > $out/pytest.txt 2>&1
  echo "pytest rc=$?" >> $out/pytest.txt
fi
for w in $wls; do
  for m in "" "--fast"; do
    tag=$w${m:+_fast}
    timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline $m \
      > $out/bench_$tag.json 2> $out/bench_$tag.err
  done
done
python tools/brief.py $out > $out/brief.txt 2>&1
cat $out/brief.txt

#!/bin/bash
# compute-sanitizer over the small parity shapes
out=${1:-gpurun_out/r02s}
mkdir -p $out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > $out/$tool.log 2>&1
  echo "$tool rc=$?" >> $out/$tool.log
  tail -4 $out/$tool.log
done
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_small.py large > $out/memcheck_large.log 2>&1
echo "memcheck large rc=$?" >> $out/memcheck_large.log
tail -4 $out/memcheck_large.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_small.py large > $out/racecheck_large.log 2>&1
echo "racecheck large rc=$?" >> $out/racecheck_large.log
tail -4 $out/racecheck_large.log

#!/bin/bash
# final-state check: full GPU suite, smoke, bench lines of the configs touched after the main evidence run
out=${1:-gpurun_out/r02f}
mkdir -p $out
timeout 1800 python -m pytest tests -q -m gpu --durations=5 > $out/pytest.txt 2>&1
echo "pytest rc=$?" >> $out/pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1
python bench.py > $out/bench_c3.json 2> $out/bench_c3.err
for w in c1 c2v c2w c0; do
  python bench.py --workload $w --steps 5 --warmup 3 > $out/bench_$w.json 2> $out/bench_$w.err
done
python bench.py --workload c4 --reps 50 > $out/bench_c4.json 2> $out/bench_c4.err
python tools/brief.py $out > $out/brief.txt 2>&1
tail -3 $out/pytest.txt; tail -3 $out/smoke.txt; grep -E "^bench" $out/brief.txt
python -c "
import json; j=json.loads(open('$out/bench_c4.json').read().strip().splitlines()[-1]); print({k:(v['ms_per_launch'],v['frac']) for k,v in j['kernels'].items()})"

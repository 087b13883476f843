bash tools/r02_slices.sh gpurun_out/r02slices
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for w in c1 c2v c0; do
python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-extras > /tmp/b.json 2>/dev/null; python -c "
import json; j=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$w', round(j['ms_per_step'],2))"
done

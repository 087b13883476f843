timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for w in c2w c0 c1 c3; do
python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-extras > /tmp/b.json 2>/dev/null; python -c "
import json; j=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$w', round(j['ms_per_step'],2), {k:round(v['ms'],2) for k,v in j['breakdown_one_solve'].items()})"
done
python tools/tail_trace.py 2 W 2>&1 | tail -15

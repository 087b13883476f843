for e in 0 1; do
for w in c2v; do
PMG_EXACT_MODE=$e python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-extras > /tmp/b.json 2>/dev/null; python -c "
import json; j=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('mode $e $w', round(j['ms_per_step'],2), {k:v['ms'] for k,v in j['breakdown_one_solve'].items()}, {k:v['ms_per_launch'] for k,v in j['kernels_finest_level'].items()})"
done; done
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_large.py -q -m gpu -x 2>&1 | tail -2

for l in libpolarmg_b200.so libpolarmg_b200_t3.so libpolarmg_b200_t6.so; do
PMG_LIB=$PWD/paper_2507_03812_b200/lib/$l python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --no-extras > /tmp/b.json 2>/dev/null; python -c "
import json; j=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$l', round(j['ms_per_step'],2), {k:v['ms'] for k,v in j['breakdown_one_solve'].items()}, {k:v['ms_per_launch'] for k,v in j['kernels_finest_level'].items()})"
done
PMG_PROLONG_LINES=0 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --no-extras > /tmp/b.json 2>/dev/null; python -c "
import json; j=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('nolines', round(j['ms_per_step'],2), {k:v['ms'] for k,v in j['breakdown_one_solve'].items()})"
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2

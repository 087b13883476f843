timeout 900 python -m pytest tests/test_gpu_configs.py::test_config3_all_sections tests/test_gpu_configs.py::test_config3_sections_fast_mode tests/test_gpu_determinism.py tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
for m in "" "--fast"; do
python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline $m > /tmp/b.json 2>/dev/null; python -c "
import json; j=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('c3 $m', round(j['ms_per_step'],2), {k:(v['ms_per_launch'],v['frac']) for k,v in j['kernels_finest_level'].items()}, {k:v['ms'] for k,v in j['breakdown_one_solve'].items()})"
done

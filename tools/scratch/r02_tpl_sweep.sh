PMG_TPL=0 timeout 900 python -m pytest tests/test_gpu_configs.py::test_config3_all_sections tests/test_gpu_determinism.py -q -m gpu -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_configs.py::test_config3_all_sections -q -m gpu -x 2>&1 | tail -2
for v in "PMG_TPL=0" "PMG_TPL=1" ; do
for m in "" "--fast"; do
env $v python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline $m > /tmp/b.json 2>/dev/null; python -c "
import json; j=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$v $m', round(j['ms_per_step'],2), j['kernels_finest_level']['radial']['ms_per_launch'], j['breakdown_one_solve']['radial'])"
done; done

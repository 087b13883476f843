for l in libpolarmg_b200.so libpolarmg_b200_ex8.so; do
for w in c1 c2v c0; do
PMG_LIB=$PWD/paper_2507_03812_b200/lib/$l python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-extras > /tmp/b.json 2>/dev/null; python -c "
import json; j=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$l $w', round(j['ms_per_step'],2), {k:v['ms'] for k,v in j['breakdown_one_solve'].items()})"
done; done
PMG_LIB=$PWD/paper_2507_03812_b200/lib/libpolarmg_b200_ex8.so timeout 900 python -m pytest tests/test_gpu_configs.py -q -m gpu -x -k "config_solve and not fast" 2>&1 | tail -2

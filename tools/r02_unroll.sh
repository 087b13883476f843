for l in libpolarmg_b200.so libpolarmg_b200_u3.so libpolarmg_b200_u4.so; do
PMG_LIB=$PWD/paper_2507_03812_b200/lib/$l python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline > /tmp/b.json 2>/dev/null; python -c "
import json; j=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$l', round(j['ms_per_step'],2), {k:(v['ms_per_launch'],v['frac']) for k,v in j['kernels_finest_level'].items()})"
done

for v in "X=0" "PMG_FUSED_SMALL_T=64" "PMG_FUSED_SMALL_T=256" "PMG_FUSED_SMOOTH=0" "PMG_COARSE_SMEM=120000" "PMG_COARSE_SMEM=60000" "PMG_ROWS_NODES=1200000" "PMG_ROWS_NODES=0" "PMG_MID_NODES=20000"; do
for w in c1 c0; do
env $v python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-extras > /tmp/b.json 2>/dev/null; python -c "
import json; j=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$v $w', round(j['ms_per_step'],3), {k:round(v['ms'],2) for k,v in j['breakdown_one_solve'].items()})"
done; done

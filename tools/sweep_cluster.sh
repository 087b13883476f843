for rows in 900 1200 1800; do for k in 4 8; do
echo -n "rows=$rows K=$k: "; PMG_LINE_CLUSTER_ROWS=$rows PMG_RADIAL_K=$k python bench.py --workload c4 --reps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:(v['ms_per_launch'],v['frac']) for k,v in d['kernels'].items() if k=='radial'})"
done; done
for rows in 1024 2048 4096; do echo -n "circle rows=$rows: "; PMG_CIRCLE_CLUSTER_ROWS=$rows python bench.py --workload c4 --reps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:(v['ms_per_launch'],v['frac']) for k,v in d['kernels'].items() if k=='circle'})"; done

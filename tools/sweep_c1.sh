run() { echo -n "$1: "; env $2 python bench.py --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3))"; }
run default ""
run circ512 "PMG_CIRCLE_CLUSTER_ROWS=512"
run rad2 "PMG_RADIAL_CL_MIN=512 PMG_LINE_CLUSTER_ROWS=450"
run both "PMG_CIRCLE_CLUSTER_ROWS=512 PMG_RADIAL_CL_MIN=512 PMG_LINE_CLUSTER_ROWS=450"
run rad3 "PMG_RADIAL_CL_MIN=256 PMG_LINE_CLUSTER_ROWS=300"
run circ256 "PMG_CIRCLE_CLUSTER_ROWS=256"

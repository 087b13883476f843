#!/bin/bash
# Give-operator roofline at 4097x4096: bench line, then ncu FP64-instruction and DRAM counts
out=${1:-gpurun_out/r02g}
mkdir -p $out
python bench.py --workload give --reps 20 > $out/bench_give_pre.json 2> $out/bench_give.err
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
ncu --metrics $M --clock-control none -k regex:"k_apply|k_circle|k_radial" --csv --log-file $out/give_metrics.csv \
    python bench.py --workload give --reps 1 > $out/give_ncu.log 2>&1
python tools/give_flops.py $out/give_metrics.csv 4097 4096 652 profiles/give_flops.json > $out/give_flops.md 2>&1
cat $out/give_flops.md
cp profiles/give_flops.json $out/
python bench.py --workload give --reps 20 > $out/bench_give.json 2>> $out/bench_give.err
cat $out/bench_give.json

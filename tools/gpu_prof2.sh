#!/bin/bash
# launch list + full ncu capture of two K2 launches: u=2 group 0 (-s 2) and a late one (-s 150)
TAG=${1:-run}
OUT=gpurun_out
mkdir -p $OUT
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/launches_$TAG.csv python bench.py --profile > $OUT/ncu_launch_$TAG.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_dp_step -s 2 -c 1 -o $OUT/prof_u2_$TAG \
    python bench.py --profile > $OUT/ncu_u2_$TAG.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_dp_step -s 150 -c 2 -o $OUT/prof_late_$TAG \
    python bench.py --profile > $OUT/ncu_late_$TAG.log 2>&1
echo done

#!/bin/bash
# ncu only: launch list of one device pass + full capture of a few K2 launches.
# usage (under gpurun): bash tools/gpu_prof.sh tag
TAG=${1:-run}
OUT=gpurun_out
mkdir -p $OUT
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/launches_$TAG.csv python bench.py --profile > $OUT/ncu_launch_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_dp_(classify|rounds)" -s 40 -c 4 -o $OUT/prof_k2_$TAG \
    python bench.py --profile > $OUT/ncu_full_$TAG.log 2>&1
echo done

#!/bin/bash
# One GPU round trip: parity tests, bench, ncu launch list (one device pass) + full capture of K2.
# usage (under gpurun): bash tools/gpu_cycle.sh [tag] [extra bench args]
TAG=${1:-run}
shift
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 3 "$@" > $OUT/bench_$TAG.log 2>&1; echo "bench rc=$?" >> $OUT/bench_$TAG.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/launches_$TAG.csv python bench.py --profile > $OUT/ncu_launch_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_dp_(classify|rounds|tile)" -s 40 -c 6 -o $OUT/prof_k2_$TAG \
    python bench.py --profile > $OUT/ncu_full_$TAG.log 2>&1
tail -2 $OUT/pytest_gpu_$TAG.log

#!/bin/bash
# Quick GPU round trip: parity tests + bench only.  usage (under gpurun): bash tools/gpu_quick.sh tag [bench args]
TAG=${1:-run}
shift
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 3 "$@" > $OUT/bench_$TAG.log 2>&1; echo "bench rc=$?" >> $OUT/bench_$TAG.log
tail -2 $OUT/pytest_gpu_$TAG.log

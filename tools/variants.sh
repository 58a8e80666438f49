#!/bin/bash
# A/B of env-var variants on the sweep bench (GPU box): bash tools/variants.sh TAG "ENV=.. ENV2=.." "ENV=.." ...
TAG=$1
shift
mkdir -p gpurun_out
i=0
for v in "$@"; do
  env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/var_${TAG}_$i.log 2>&1
  echo "$v" >> gpurun_out/var_${TAG}_$i.log
  i=$((i+1))
done

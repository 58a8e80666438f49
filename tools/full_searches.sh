# full planner searches through bench.py (GPU box): one JSON line per workload into gpurun_out/fs_<name><suffix>.json
# usage: bash tools/full_searches.sh [suffix]   (env vars pass through to bench.py)
SUF=${1:-}
for w in gpt96 gpt96-bmw swin-bmw vit-bmw bert t5-16; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/fs_$w$SUF.log 2>&1
  tail -1 gpurun_out/fs_$w$SUF.log > gpurun_out/fs_$w$SUF.json
done

# full planner searches through bench.py (GPU box): one JSON line per workload into gpurun_out/fs_<name>.json
for w in gpt96 gpt96-bmw swin-bmw vit-bmw bert t5-16; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/fs_$w.log 2>&1
  tail -1 gpurun_out/fs_$w.log > gpurun_out/fs_$w.json
done

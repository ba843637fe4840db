#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for s in pull_wm; do
  timeout 600 python bench.py --steps 3 --warmup 3 --schedule $s --no-e2e --no-cpu > gpurun_out/bench_$s.json 2> gpurun_out/bench_$s.err
  timeout 600 python bench.py --steps 3 --warmup 3 --schedule $s --fp32-contrib --no-e2e --no-cpu > gpurun_out/bench_${s}32.json 2> gpurun_out/bench_${s}32.err
  timeout 600 python bench.py --steps 3 --warmup 3 --schedule $s --permute --no-e2e --no-cpu > gpurun_out/bench_${s}_perm.json 2> gpurun_out/bench_${s}_perm.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pr_pull -s 5 -c 1 -o gpurun_out/prof_pull python bench.py --steps 1 --warmup 1 --schedule pull_wm --no-e2e --no-cpu > gpurun_out/ncu_pull.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_edge_blocked -s 2 -c 1 -o gpurun_out/prof_eb python bench.py --steps 1 --warmup 1 --schedule eb --no-e2e --no-cpu > gpurun_out/ncu_eb.log 2>&1

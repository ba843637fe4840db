#!/bin/bash
# First GPU session: tests, smoke, PR schedule exploration at C5.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1; free -g >> gpurun_out/nvsmi.txt; nproc >> gpurun_out/nvsmi.txt
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.txt 2>&1
for s in eb edge pull push; do
  timeout 600 python bench.py --steps 3 --warmup 3 --schedule $s --no-e2e --no-cpu > gpurun_out/bench_$s.json 2> gpurun_out/bench_$s.err
done
timeout 600 python bench.py --steps 3 --warmup 3 --schedule pull --fp32-contrib --no-e2e --no-cpu > gpurun_out/bench_pull32.json 2> gpurun_out/bench_pull32.err
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err

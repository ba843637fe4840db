#!/bin/bash
# Round-1 re-entry: state of HEAD on a B200 (tests, smoke, bench f64/f32, launch list).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --steps 3 --warmup 3 --fp32-contrib --no-e2e --no-cpu > gpurun_out/bench_eb32.json 2> gpurun_out/bench_eb32.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_eb64.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/launches_eb64.log 2>&1

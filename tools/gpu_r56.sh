#!/bin/bash
# final round-1 validation and bench lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/f_c5.json 2> gpurun_out/f_c5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err
timeout 600 python bench.py --config c2 --check > gpurun_out/f_c2.json 2> gpurun_out/f_c2.err
timeout 600 python bench.py --config c3 --steps 2 --check > gpurun_out/f_c3.json 2> gpurun_out/f_c3.err
timeout 1200 python bench.py --config c4 --steps 2 --check > gpurun_out/f_c4.json 2> gpurun_out/f_c4.err

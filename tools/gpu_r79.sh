#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout=120 --timeout-method=thread > gpurun_out/r79_tests.txt 2>&1
timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > gpurun_out/r79_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r79_c5.json 2> gpurun_out/r79_c5.err
timeout 300 python bench.py --impl reference > gpurun_out/r79_ref.json 2> gpurun_out/r79_ref.err

#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python tools/e2e_breakdown.py > gpurun_out/e2e_default.txt 2>&1
timeout 900 python bench.py > gpurun_out/r63_c5.json 2> gpurun_out/r63_c5.err
timeout 900 python bench.py --fp32-contrib > gpurun_out/r63_c5_32.json 2> gpurun_out/r63_c5_32.err
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout=900 --timeout-method=thread > gpurun_out/r63_tests.txt 2>&1
python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > gpurun_out/r63_smoke.txt 2>&1

#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout=300 --timeout-method=thread > gpurun_out/r77_tests.txt 2>&1
timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > gpurun_out/r77_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r77_c5.json 2> gpurun_out/r77_c5.err
timeout 600 python bench.py --config c2 --check > gpurun_out/r77_c2.json 2> gpurun_out/r77_c2.err
timeout 600 python bench.py --config c4 > gpurun_out/r77_c4.json 2> gpurun_out/r77_c4.err

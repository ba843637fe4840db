#!/bin/bash
# tools/sweep_c2.sh TAG "bench args" ... : C2 DO-BFS variants (16 sources), compact lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=$1; shift
for c in "$@"; do
  timeout 900 python bench.py --config c2 --sources 16 $c > gpurun_out/${tag}_tmp.json 2> gpurun_out/${tag}_tmp.err
  python - "$c" gpurun_out/${tag}_tmp.json >> gpurun_out/${tag}_c2sweep.txt <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print("%-50s %7.1f GTEPS hmean  median %.3f ms/source  ok %s" % (sys.argv[1], d["value"], d["ms_per_step"],
          d["parity"]["ok"]))
except Exception as e:
    print("%-50s FAILED %s" % (sys.argv[1], e))
PY
done

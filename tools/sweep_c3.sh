#!/bin/bash
# tools/sweep_c3.sh TAG DELTAS "ENV=.. ENV2=.." ... : C3 (fused SSSP, VERTEX_BASED) per env case
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=$1; deltas=$2; shift 2
for c in "$@"; do
  for d in $deltas; do
    env $c timeout 300 python bench.py --config c3 --lb VERTEX_BASED --delta $d --steps 3 --warmup 1 \
      > gpurun_out/${tag}_tmp.json 2> gpurun_out/${tag}_tmp.err
    python - "$c" $d gpurun_out/${tag}_tmp.json >> gpurun_out/${tag}_c3sweep.txt <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
    s = list(d["config"]["delta_sweep"].values())[0]
    print("%-40s delta %6s  %8.2f ms  rounds %6d  traversed %6.2fxA  ok %s" % (
        sys.argv[1], sys.argv[2], d["ms_per_step"], s["rounds"], s["edges_traversed"] / d["config"]["arcs"],
        d["parity"]["ok"]))
except Exception as e:
    print("%-40s delta %s FAILED %s" % (sys.argv[1], sys.argv[2], e))
PY
  done
done

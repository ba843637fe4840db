#!/bin/bash
# Env-knob sweep of the C5 PageRank step: tools/sweep_pr.sh TAG "VAR=a VAR2=b" "VAR=c" ...
# Each case prints one compact line (GTEPS, hot-kernel frac, iteration frac).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=$1; shift
for c in "$@"; do
  env $c timeout 600 python bench.py --no-e2e --no-cpu --no-sub --no-parity --steps 3 --warmup 3 \
    > gpurun_out/${tag}_tmp.json 2> gpurun_out/${tag}_tmp.err
  python - "$c" gpurun_out/${tag}_tmp.json >> gpurun_out/${tag}_sweep.txt <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print("%-40s %7.1f GTEPS  ms/step %7.2f  hot %.2f ms frac %.3f  edge %.3f  iter %.3f  sm %s" % (
        sys.argv[1], d["value"], d["ms_per_step"], r["avg_launch_ms"], r["frac"], r["edge_phase"]["frac"],
        r["iteration_frac"], d["clocks"]["sm_mhz"]))
except Exception as e:
    print("%-40s FAILED %s" % (sys.argv[1], e))
PY
done

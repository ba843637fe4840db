#!/bin/bash
# tools/sweep_c4.sh TAG "ENV=.." ... : C4 (CC per load balancer + BC) per env case, compact lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=$1; shift
for c in "$@"; do
  env $c timeout 900 python bench.py --config c4 --steps 3 --warmup 1 > gpurun_out/${tag}_tmp.json 2> gpurun_out/${tag}_tmp.err
  python - "$c" gpurun_out/${tag}_tmp.json >> gpurun_out/${tag}_c4sweep.txt <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    cfg = d["config"]
    cc = " ".join("%s %.1f" % (k, v["gteps"]) for k, v in cfg["cc"].items())
    bc = " ".join("%s %.1f" % (k, v["gteps"]) for k, v in cfg["bc"].items())
    print("%-24s CC[%s] BC[%s] prep %.0f ms e2e %.1f ok %s" % (sys.argv[1], cc, bc, cfg.get("relabel_prep_ms", 0),
          d["e2e"]["value"], d["parity"]["ok"]))
except Exception as e:
    print("%-24s FAILED %s" % (sys.argv[1], e))
PY
done

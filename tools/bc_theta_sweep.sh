cd $GRAFT_REPO_ROOT
for t in 0.001 0.003 0.01 0.03 0.1; do
  timeout 900 python bench.py --config c4 --lbs ETWC,HYBRID --bc-theta $t --steps 1 --warmup 1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('theta $t', round(d['config']['bc']['HYBRID']['gteps'],1), d['parity']['ok'])" >> gpurun_out/bct_sweep.txt
done

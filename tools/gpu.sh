#!/bin/bash
# One runner for every gpurun session (replaces the per-session gpu_r*.sh
# scripts of round 1, which live in git history at commit 5acd546).
#
#   gpurun --timeout T -- 'bash tools/gpu.sh TAG STEP [STEP ...]'
#
# Each STEP writes gpurun_out/TAG_<name>.{txt,json,err}; steps:
#   host               nproc / free -g / nvidia-smi -L
#   tests[=EXPR]       pytest -m gpu (optionally -k EXPR)
#   smoke              __graft_entry__.smoke()
#   bench[=ARGS]       python bench.py ARGS (default: the driver's default run)
#   launches[=ARGS]    ncu launch list (gpu__time_duration) of bench.py ARGS
#   launchesw[=ARGS]   same, --cache-control none (warm caches between launches)
#   ncu=REGEX@ARGS     ncu --set full of the first launch matching REGEX
#   py=SCRIPT@ARGS     python SCRIPT ARGS
# Arguments use ',' for spaces (bench=--config,c2,--check).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=$1; shift
for step in "$@"; do
  name=${step%%=*}; arg=""
  [[ "$step" == *=* ]] && arg=${step#*=}
  arg=${arg//,/ }
  out=gpurun_out/${tag}_${name}
  case $name in
    host)
      { nproc; free -g; nvidia-smi -L; nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv; } > $out.txt 2>&1 ;;
    tests)
      k=(); [ -n "$arg" ] && k=(-k "$arg")
      timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout=600 \
        --timeout-method=thread "${k[@]}" > $out.txt 2>&1; echo "rc=$?" >> $out.txt ;;
    smoke)
      timeout 600 python -c 'import __graft_entry__ as g; g.smoke()' > $out.txt 2>&1; echo "rc=$?" >> $out.txt ;;
    bench)
      timeout 1800 python bench.py $arg > $out.json 2> $out.err; echo "rc=$?" >> $out.err ;;
    launches)
      timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file $out.csv python bench.py $arg > $out.txt 2>&1 ;;
    launchesw)
      timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --cache-control none --csv --log-file $out.csv python bench.py $arg > $out.txt 2>&1 ;;
    ncu)
      re=${arg%%@*}; a=${arg#*@}
      timeout 1800 ncu --set full --clock-control none --import-source on -k "regex:$re" -c 1 \
        -o $out python bench.py $a > $out.txt 2>&1
      # the binary report may not survive the trip back: summarise it here
      ncu -i $out.ncu-rep --page raw --csv > $out.raw.csv 2>&1
      python tools/ncu_summary.py $out.summary.txt $out.ncu-rep > /dev/null 2>&1 ;;
    py)
      s=${arg%%@*}; a=""; [[ "$arg" == *@* ]] && a=${arg#*@}
      timeout 1800 python $s $a > $out.txt 2>&1; echo "rc=$?" >> $out.txt ;;
    *) echo "unknown step $name" >&2 ;;
  esac
done

#!/bin/bash
# compute-sanitizer evidence: memcheck over the small-graph GPU tests,
# racecheck/synccheck on the shared-memory kernels (ETWC, PR hot-segment cache).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --error-exitcode 99 --print-limit 20 python -m pytest tests/test_gpu_engine.py tests/test_gpu_graph.py "tests/test_gpu_algos.py::test_bfs_golden" "tests/test_gpu_algos.py::test_cc_golden" "tests/test_gpu_algos.py::test_sssp_golden" "tests/test_gpu_algos.py::test_bc_golden" "tests/test_gpu_pagerank.py::test_pagerank_every_schedule_matches_oracle" "tests/test_gpu_pagerank.py::test_pagerank_edge_blocking_edge_cases" "tests/test_gpu_dist.py::test_bfs_virtual_ranks_levels_and_tree" -m gpu -q -x -p no:cacheprovider > gpurun_out/sanitizer_memcheck.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_memcheck.txt
timeout 900 $CS --tool racecheck --error-exitcode 99 --print-limit 20 python -m pytest "tests/test_gpu_pagerank.py::test_pagerank_edge_blocking_matches_oracle" "tests/test_gpu_algos.py::test_etwc_hub_pass_bfs_cc" -m gpu -q -x -p no:cacheprovider > gpurun_out/sanitizer_racecheck.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_racecheck.txt
timeout 900 $CS --tool synccheck --error-exitcode 99 --print-limit 20 python -m pytest "tests/test_gpu_pagerank.py::test_pagerank_edge_blocking_matches_oracle" "tests/test_gpu_algos.py::test_bfs_every_schedule" -m gpu -q -x -p no:cacheprovider > gpurun_out/sanitizer_synccheck.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_synccheck.txt

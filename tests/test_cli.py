"""The schedge-compatible CLI: parser surface on CPU, commands on the GPU."""

import json
import os
import subprocess
import sys

import pytest

from paper_2012_07990_b200 import cli
from tests.conftest import ROOT


def test_parser_matches_reference_surface():
    p = cli.build_parser()
    a = p.parse_args(["run", "pr", "g.txt", "--schedule", "s.sched", "--out", "x",
                      "--sched-arg", "0=0.2", "--max-iters", "20"])
    assert a.fn is cli.cmd_run and a.out == "x" and a.sched_arg == ["0=0.2"]
    a = p.parse_args(["tune", "bfs", "g.txt", "--budget", "3", "--strategy", "random"])
    assert a.fn is cli.cmd_tune and a.trials == "trials.csv" and a.out == "best.sched"
    a = p.parse_args(["convert", "g.txt", "--out", "g.blk", "--block", "64"])
    assert a.fn is cli.cmd_convert
    assert cli._canonical_algo("pr") == "pagerank" and cli._canonical_algo("sssp_delta") == "sssp"
    with pytest.raises(SystemExit):
        cli._canonical_algo("nope")


def test_list_labels_runs_without_a_gpu():
    out = subprocess.run([sys.executable, "-m", "paper_2012_07990_b200", "list-labels", "--space"],
                         cwd=ROOT, capture_output=True, text=True, check=True).stdout
    assert "raw combinations:   2016" in out and "valid combinations: 1152" in out


@pytest.mark.gpu
def test_cli_run_bench_verify_convert(tmp_path):
    edges = tmp_path / "g.txt"
    edges.write_text("# tiny\n0 1\n1 2\n2 0\n2 3\n")
    prefix = str(tmp_path / "run")
    assert cli.main(["run", "bfs", str(edges), "--source", "0", "--out", prefix]) == 0
    assert open(prefix + ".values.txt").read().split() == ["0", "0", "1", "2"]
    st = json.load(open(prefix + ".stats.json"))
    assert st["algorithm"] == "bfs" and st["rounds"] >= 3
    assert cli.main(["bench", "pr", "rmat:10:8:3", "--max-iters", "5"]) == 0
    assert cli.main(["verify", "cc", "rmat:9:8:2", "--samples", "4"]) == 0
    out = str(tmp_path / "g.blk")
    assert cli.main(["convert", str(edges), "--out", out, "--block", "2"]) == 0
    from paper_2012_07990_b200.blocking import load_blocked
    bg = load_blocked(out)
    assert bg.num_edges == 4 and bg.segment_start[-1] == 4
    assert cli.main(["run", "sssp", "grid:8", "--out", prefix, "--delta", "64"]) == 0

"""The GPU CLI (paper_2206_05543_b200.cli): argument surface and RunRecord schema of the
reference CLI's solve/bench (reference cli.py:18-52, :215-266, :326-377, :416-447), and the
example right-hand sides against the reference's problems.py when it is importable here."""
import json
import os
import sys

import numpy as np
import pytest

from paper_2206_05543_b200 import cli, problems

REF = "/root/reference/pkg/src"


def test_parser_mirrors_reference_solve_and_bench():
    p = cli.build_parser()
    a = p.parse_args(["solve", "--example", "3", "--N", "16", "--smoother", "m7"])
    assert (a.cycle, a.nu1, a.nu2, a.seed, a.tol, a.max_iters, a.format) == ("w", 1, 0, 0, 1e-10, 100, "csv")
    a = p.parse_args(["bench"])
    assert (a.examples, a.Ns, a.cycles, a.max_iters) == ("1", "64,128,256", "w1+0,v1+1", 100)
    with pytest.raises(SystemExit):
        p.parse_args(["solve", "--example", "4", "--N", "16", "--smoother", "m7"])
    assert cli.BENCH_COLUMNS[0] == "example" and cli.SCHEMA_VERSION == 1


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
@pytest.mark.parametrize("k,N", [(1, 16), (2, 12), (3, 8)])
def test_rhs_matches_reference(k, N):
    sys.path.insert(0, REF)
    try:
        from spaimg import problems as rp
        ref = rp.assemble_rhs(rp.example(k), N).values
    finally:
        sys.path.remove(REF)
    assert np.array_equal(problems.assemble_rhs(problems.example(k), N).values, ref)


@pytest.mark.gpu
def test_cli_solve_and_bench_on_gpu(tmp_path):
    out = tmp_path / "rec.json"
    rc = cli.main(["solve", "--example", "3", "--N", "32", "--cycle", "v", "--nu1", "1", "--nu2", "1",
                   "--smoother", "m7", "--out", str(out), "--format", "json"])
    rec = json.load(open(out))
    assert rc == 0 and rec["command"] == "solve" and rec["schema_version"] == 1
    assert rec["outputs"]["converged"] and rec["outputs"]["error_inf"] < 1e-2
    csvp = tmp_path / "bench.csv"
    rc = cli.main(["bench", "--examples", "1", "--Ns", "32,64", "--cycles", "v1+1", "--out", str(csvp)])
    lines = open(csvp).read().strip().splitlines()
    assert rc == 0 and lines[0].split(",") == cli.BENCH_COLUMNS and len(lines) == 1 + 2 * 3

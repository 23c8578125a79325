"""The tileinv CLI (cli.py; SPEC.md module `cli`): analysis commands and
validation exits on CPU, invert / bench on the B200."""

import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1002_4057_b200 import _native
from paper_1002_4057_b200.cli import main

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_table_exit_codes(capsys):
    # SPEC.md cmd_table: nonzero exit on any mismatch; the pipelined rows of the
    # reference do not follow Table 1 (SURVEY.md finding 6)
    assert main(["table", "--t-min", "2", "--t-max", "8"]) == 3
    out = capsys.readouterr().out
    assert out.startswith("variant,t,measured,formula,match\n")
    assert "step3/out,4,4,4,true" in out
    assert main(["table", "--allow-mismatch"]) == 0
    assert main(["table", "--t-min", "1"]) == 2


def test_dag_export(tmp_path, capsys):
    # SPEC.md cmd_dag examples: step 3 in-place t=4 -> 20 nodes, critical path 10;
    # out-of-place -> 4; full pipeline t=2 in-place -> 9 (9t-9)
    out = tmp_path / "s3.dot"
    assert main(["dag", "--t", "4", "--step", "3", "--out", str(out)]) == 0
    dot = out.read_text()
    assert dot.startswith("digraph") and dot.count("[label=") - dot.count("->") == 20
    assert "critical path 10 tasks" in capsys.readouterr().out
    assert main(["dag", "--t", "4", "--step", "3", "--placement", "out", "--out", str(out)]) == 0
    assert "critical path 4 tasks" in capsys.readouterr().out
    assert main(["dag", "--t", "2", "--loops", "UDU"]) == 0
    assert "critical path 11 tasks" in capsys.readouterr().err


def test_validation_exits():
    assert main(["invert", "--n", "300", "--b", "200"]) == 2  # SPEC.md: divisibility error
    assert main(["invert", "--n", "400", "--b", "200", "--loops", "UXU"]) == 2
    assert main(["invert", "--n", "400", "--b", "200", "--workers", "0"]) == 2
    assert main(["bench", "--n", "300", "--b", "200"]) == 2
    assert main(["invert", "--input", "/nonexistent/a.csv", "--b", "2"]) == 4


def test_module_entry_point():
    r = subprocess.run([sys.executable, "-m", "paper_1002_4057_b200", "table", "--allow-mismatch", "--t-max", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.splitlines()[0] == "variant,t,measured,formula,match"


def test_invert_without_device_fails_loudly():
    if _native.device_count() > 0:
        pytest.skip("a B200 is present")
    assert main(["invert", "--n", "400", "--b", "200"]) == 1


@pytest.mark.gpu
def test_invert_and_bench_on_gpu(tmp_path, capsys):
    # SPEC.md cmd_invert examples: n=400 b=200 residual <= 1e-9 n, exit 0; t=1 chain
    assert main(["invert", "--n", "400", "--b", "200"]) == 0
    assert "residual=" in capsys.readouterr().out
    assert main(["invert", "--n", "200", "--b", "200", "--placement", "out", "--no-pipeline"]) == 0
    a = np.eye(6) * 4.0
    a[5, 5] = -1.0
    f = tmp_path / "a.csv"
    np.savetxt(f, a, delimiter=",")
    assert main(["invert", "--input", str(f), "--b", "3"]) == 3  # POTRF failure reported
    assert "inversion failed" in capsys.readouterr().err
    csv = tmp_path / "b.csv"
    assert main(["bench", "--n", "512", "--b", "128", "--placement", "in", "out", "--both-pipelining",
                 "--out", str(csv)]) == 0
    rows = csv.read_text().strip().split("\n")
    assert rows[0] == "variant,n,b,workers,loops,pipelined,time_s,gflops" and len(rows) == 5
    for r in rows[1:]:
        v, n, b, w, loops, pipe, ts, gf = r.split(",")
        assert v in ("in", "out") and n == "512" and float(ts) > 0 and float(gf) > 0

"""CLI hook, host side (no GPU): compare consumes the REFERENCE's own solve
summaries (tests/golden/cli_ref, written by the reference's mpcg solve), the
reference's exit codes for usage and I/O errors."""
import json
import os

from conftest import ROOT

REF = os.path.join(ROOT, "tests", "golden", "cli_ref")


def test_compare_reference_summaries(tmp_path, capsys):
    from paper_2407_15973_b200 import cli
    out = tmp_path / "cmp.json"
    rc = cli.main(["compare", os.path.join(REF, "uniform.summary.json"),
                   os.path.join(REF, "fixed-low.summary.json"), "--out", str(out)])
    assert rc == 0
    res = json.loads(out.read_text())
    assert (res["iterations_a"], res["iterations_b"]) == (21, 28)
    assert res["iteration_ratio"] == 28 / 21
    assert res["backend_a"] == "numba"
    assert "iterations" in capsys.readouterr().out


def test_cli_error_codes(tmp_path):
    from paper_2407_15973_b200 import cli
    assert cli.main(["compare", str(tmp_path / "missing.json"), str(tmp_path / "x.json")]) == 3
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert cli.main(["compare", str(bad), str(bad)]) == 2
    assert cli.main(["solve", "--out", str(tmp_path / "o")]) == 2           # no problem
    assert cli.main(["solve", "--problem", "const", "--out", str(tmp_path / "o")]) == 2  # no --n
    assert cli.main(["solve", "--problem", "const", "--n", "4", "--rhs", "zeros",
                     "--out", str(tmp_path / "o")]) == 2
    assert cli.main(["solve", "--matrix", str(tmp_path / "none.mtx"), "--out", str(tmp_path / "o")]) == 3
    assert cli.main(["bogus"]) == 2

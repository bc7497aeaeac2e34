"""CLI hook on the GPU: ``solve`` writes the reference's trace / summary
formats (so the reference's ``mpcg compare`` can read them) and ``compare``
takes a summary of each backend (tests/golden/cli_ref: the reference's own
``mpcg solve`` of the same problem)."""
import json
import os

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
REF = os.path.join(ROOT, "tests", "golden", "cli_ref")


def test_solve_matches_reference_summary_and_compares(cuda, tmp_path):
    from paper_2407_15973_b200 import cli
    from paper_2407_15973_b200.solver import read_trace_csv
    out = tmp_path / "gpu"
    rc = cli.main(["solve", "--problem", "dis", "--n", "10", "--s", "100", "--nb", "8",
                   "--policy", "uniform", "--policy", "fixed-low", "--true-every", "5",
                   "--out", str(out)])
    assert rc == 0
    for pol in ("uniform", "fixed-low"):
        mine = json.loads((out / f"{pol}.summary.json").read_text())
        ref = json.loads(open(os.path.join(REF, f"{pol}.summary.json")).read())
        assert set(ref) <= set(mine)                       # every key the reference writes
        assert mine["problem"] == ref["problem"]           # so either compare accepts the pair
        assert mine["preconditioner"] == ref["preconditioner"] and mine["solve"] == ref["solve"]
        assert (mine["backend"], mine["reduction_mode"]) == ("b200", "tree")
        assert abs(mine["iterations"] - ref["iterations"]) <= 2
        tr = read_trace_csv(out / mine["trace_file"])
        assert len(tr) == mine["iterations"]
        cmp_json = tmp_path / f"cmp-{pol}.json"
        assert cli.main(["compare", os.path.join(REF, f"{pol}.summary.json"),
                         str(out / f"{pol}.summary.json"), "--out", str(cmp_json)]) == 0
        res = json.loads(cmp_json.read_text())
        assert res["divergence_iteration"] is None         # same residual history (dot order aside)
        assert res["backend_b"] == "b200"


def test_solve_bench_config(cuda, tmp_path):
    from paper_2407_15973_b200 import cli
    rc = cli.main(["solve", "--bench-config", "c2", "--n", "16", "--out", str(tmp_path)])
    assert rc == 0
    s = json.loads((tmp_path / "fixed-low.summary.json").read_text())
    assert s["converged"] and s["problem"]["bench_config"] == "c2"
    assert s["preconditioner"]["nb"] == 16 ** 3 // 64

"""Suite harness + CLI (paper_2312_14832_b200/suite.py, cli.py) against the
reference's own tests (proj/tests/test_bench.cpp, acceptance.cpp C6/C7/C9).
CPU tests: SGM hand values, report formats, CLI generation and input errors.
GPU tests: RunSuite over a directory, `solve` exit codes and solution file,
byte-identical redacted reports across runs (acceptance C9)."""
import json
import math
import random

import numpy as np
import pytest

from paper_2312_14832_b200 import cli, rpdlp, suite
from paper_2312_14832_b200.rpdlp import ResidualReport, SolveResult, SolveStatus


def test_sgm_hand_values():
    assert suite.Sgm([0.0, 0.0], 10.0, 3600.0, [True, True]) == pytest.approx(0.0, abs=1e-12)
    assert suite.Sgm([10.0, 40.0], 10.0, 3600.0, [True, True]) == pytest.approx(math.sqrt(1000.0) - 10.0, rel=1e-9)
    assert suite.Sgm([5.0], 10.0, 3600.0, [True]) == pytest.approx(5.0, rel=1e-12)


def test_sgm_charges_unsolved_the_time_limit():
    solved = suite.Sgm([1.0, 2.0], 10.0, 100.0, [True, True])
    fail = suite.Sgm([1.0, 2.0], 10.0, 100.0, [True, False])
    assert fail == pytest.approx(math.sqrt(11.0 * 110.0) - 10.0, rel=1e-9)
    assert fail > solved
    assert suite.Sgm([1.0, 55.5], 10.0, 100.0, [True, False]) == pytest.approx(fail, rel=1e-12)


def test_sgm_permutation_invariant_monotone_and_errors():
    rng = random.Random(5)
    t = [rng.uniform(0, 50) for _ in range(8)]
    base = suite.Sgm(t, 10.0, 3600.0, [True] * 8)
    s = t[:]
    rng.shuffle(s)
    assert suite.Sgm(s, 10.0, 3600.0, [True] * 8) == pytest.approx(base, rel=1e-12)
    t2 = t[:]
    t2[3] += 5.0
    assert suite.Sgm(t2, 10.0, 3600.0, [True] * 8) > base
    for args in (([], 10.0, 3600.0, []), ([1.0], 10.0, 3600.0, [True, True]), ([1.0], -1.0, 3600.0, [True])):
        with pytest.raises(ValueError):
            suite.Sgm(*args)


def test_summary_json_byte_stable_under_redaction():
    s = suite.SuiteSummary(tolerance=1e-6)
    s.records = [suite.BenchRecord("a.mps", "Optimal", 0.123, iterations=42),
                 suite.BenchRecord("b.mps", "TimeLimit", 0.456)]
    s.sgm10, s.solved_count = 1.5, 1
    red = suite.SummaryToJson(s, True)
    assert red["records"][0]["solve_seconds"] == 0.0 and red["sgm10"] == 0.0
    assert red["records"][0]["iterations"] == 42
    o = suite.SuiteSummary(tolerance=1e-6, records=[suite.BenchRecord("a.mps", "Optimal", 9.9, iterations=42),
                                                     suite.BenchRecord("b.mps", "TimeLimit", 0.456)])
    o.sgm10, o.solved_count = 77.0, 1
    assert json.dumps(suite.SummaryToJson(s, True), indent=2) == json.dumps(suite.SummaryToJson(o, True), indent=2)
    assert json.dumps(suite.SummaryToJson(s), indent=2) != json.dumps(suite.SummaryToJson(o), indent=2)
    assert list(red) == ["tolerance", "delta", "time_limit", "solved_count", "sgm10", "records"]


def test_solution_json_fields():
    r = SolveResult(SolveStatus.kOptimal, np.array([0.5]), np.array([1.0]), np.array([0.0]),
                    ResidualReport(primal_obj=2.0, dual_obj=2.0), 10, 1, 0.0, 0.0)
    j = suite.SolutionToJson(r, False)
    assert j["status"] == "Optimal" and j["primal_objective"] == 2.0 and j["dual_objective"] == 2.0
    assert j["iterations"] == 10 and j["restarts"] == 1
    assert len(j["x"]) == len(j["y"]) == len(j["lambda"]) == 1
    assert {"rel_primal", "rel_dual", "rel_gap"} <= set(j["residuals"])
    jm = suite.SolutionToJson(r, True)
    assert jm["primal_objective"] == -2.0 and jm["dual_objective"] == -2.0


def test_csv_columns(tmp_path):
    s = suite.SuiteSummary(records=[suite.BenchRecord("a.mps", "Optimal", 0.5, 0.1, 0.2, 7, 1)])
    f = tmp_path / "r.csv"
    suite.WriteSummaryCsv(s, str(f))
    lines = f.read_text().splitlines()
    assert lines[0] == ("instance,status,solve_seconds,parse_seconds,scaling_seconds,iterations,restarts,"
                        "rel_primal,rel_dual,rel_gap,primal_obj")
    assert lines[1].startswith("a.mps,Optimal,0.500000,0.100000,0.200000,7,1,")


def test_cli_gen_and_input_errors(tmp_path, capsys):
    out = tmp_path / "p.mps"
    assert cli.main(["gen", "random", "--rows", "5", "--cols", "6", "--density", "0.5", "--seed", "3",
                     "--out", str(out)]) == 0
    p = rpdlp.ParseMpsFile(out)
    q = rpdlp.GenRandomLp(5, 6, 0.5, 3)
    np.testing.assert_array_equal(p.g.values, q.g.values)
    assert cli.main(["gen", "transport", "--sources", "3", "--sinks", "4", "--out", str(tmp_path / "t.mps")]) == 0
    assert cli.main(["gen", "staircase", "--stages", "2", "--rows-per-stage", "5", "--cols-per-stage", "6",
                     "--nnz-per-row", "3", "--linking-per-row", "1", "--out", str(tmp_path / "s.mps")]) == 0
    bad = tmp_path / "broken.mps"
    bad.write_text("ROWS\n N OBJ\nCOLUMNS\n")
    assert cli.main(["solve", str(bad)]) == cli.EXIT_INPUT
    assert "error:" in capsys.readouterr().err
    assert cli.main(["solve", str(tmp_path / "missing.mps")]) == cli.EXIT_INPUT


@pytest.mark.gpu
def test_run_suite_directory(tmp_path):
    """test_bench.cpp run_suite: 3 instances + a broken file + a non-MPS file."""
    for seed in (1, 2, 3):
        p = rpdlp.GenRandomLp(5, 5, 0.6, seed)
        rpdlp.WriteMpsFile(p, tmp_path / f"{p.name}_{seed}.mps")
    (tmp_path / "broken.mps").write_text("ROWS\n N OBJ\nCOLUMNS\n")
    (tmp_path / "ignored.txt").write_text("not an instance\n")
    s = suite.RunSuite(str(tmp_path), rpdlp.SolverParams(eps=1e-6))
    assert len(s.records) == 4 and s.solved_count == 3
    assert s.records[0].instance == "broken.mps" and s.records[0].status == "Error" and s.records[0].message
    assert all(r.status == "Optimal" and r.iterations > 0 for r in s.records[1:])
    assert s.sgm10 > 0.0


@pytest.mark.gpu
def test_cli_solve_and_redacted_reports_are_byte_identical(tmp_path, capsys):
    """acceptance.cpp C9: two bench runs through the CLI with --redact-timing
    produce byte-identical reports; solve writes the solution file."""
    d = tmp_path / "suite"
    d.mkdir()
    for seed in (4, 5):
        rpdlp.WriteMpsFile(rpdlp.GenRandomLp(8, 6, 0.5, seed), d / f"r{seed}.mps")
    rpdlp.WriteMpsFile(rpdlp.GenPagerank(200, 0.85, 3, 1), d / "pr.mps")
    reports = []
    for k in range(2):
        rep = tmp_path / f"rep{k}.json"
        assert cli.main(["bench", str(d), "--eps", "1e-6", "--redact-timing", "--report", str(rep),
                         "--csv", str(tmp_path / f"rep{k}.csv")]) == 0
        reports.append(rep.read_bytes())
    assert reports[0] == reports[1]
    assert json.loads(reports[0])["solved_count"] == 3
    sol = tmp_path / "sol.json"
    assert cli.main(["solve", str(d / "pr.mps"), "--eps", "1e-6", "--out", str(sol)]) == cli.EXIT_OK
    j = json.loads(sol.read_text())
    assert j["status"] == "Optimal" and abs(sum(j["x"]) - 1.0) <= 1e-4
    assert cli.main(["solve", str(d / "pr.mps"), "--eps", "1e-12", "--iter-limit", "64"]) == cli.EXIT_LIMIT
    assert "status=IterLimit" in capsys.readouterr().out


# ------------------------------------------ the C++ tool (csrc/cli_main.cpp)
def _cpp_cli():
    from pathlib import Path
    b = Path(__file__).resolve().parents[1] / "paper_2312_14832_b200" / "_build" / "rpdlp-b200"
    if not b.exists():
        pytest.skip("C++ CLI not built (nlohmann/json absent)")
    return str(b)


def test_cpp_cli_gen_matches_python_and_usage_errors(tmp_path):
    import subprocess
    cli_bin = _cpp_cli()
    a, b = tmp_path / "a.mps", tmp_path / "b.mps"
    assert subprocess.run([cli_bin, "gen", "random", "--rows", "7", "--cols", "9", "--density", "0.4", "--seed", "5",
                           "--out", str(a)]).returncode == 0
    assert cli.main(["gen", "random", "--rows", "7", "--cols", "9", "--density", "0.4", "--seed", "5",
                     "--out", str(b)]) == 0
    assert a.read_bytes() == b.read_bytes()
    assert subprocess.run([cli_bin, "gen", "pagerank", "--nodes", "50", "--out", str(a)]).returncode == 0
    assert rpdlp.ParseMpsFile(a).num_vars() == 50
    for args, code in ((["solve"], 1), (["frobnicate"], 1), (["gen", "random", "--rows", "3", "--out", "x"], 1),
                       (["solve", str(tmp_path / "missing.mps")], 3), (["solve", str(a), "--eps"], 1)):
        r = subprocess.run([cli_bin] + args, capture_output=True, text=True)
        assert r.returncode == code, (args, r.stderr)


@pytest.mark.gpu
def test_cpp_cli_solve_and_redacted_bench(tmp_path):
    """acceptance.cpp C9 through the C++ tool: two redacted bench reports are
    byte-identical; solve writes the solution file and reports limits."""
    import subprocess
    cli_bin = _cpp_cli()
    d = tmp_path / "suite"
    d.mkdir()
    for seed in (4, 5):
        rpdlp.WriteMpsFile(rpdlp.GenRandomLp(8, 6, 0.5, seed), d / f"r{seed}.mps")
    reps = []
    for k in range(2):
        rep = tmp_path / f"rep{k}.json"
        r = subprocess.run([cli_bin, "bench", str(d), "--eps", "1e-6", "--redact-timing", "--report", str(rep)],
                           capture_output=True, text=True)
        assert r.returncode == 0 and "solved=2/2" in r.stdout
        reps.append(rep.read_bytes())
    assert reps[0] == reps[1] and json.loads(reps[0])["solved_count"] == 2
    sol = tmp_path / "sol.json"
    r = subprocess.run([cli_bin, "solve", str(d / "r4.mps"), "--eps", "1e-6", "--out", str(sol)],
                       capture_output=True, text=True)
    assert r.returncode == 0 and "status=Optimal" in r.stdout
    assert json.loads(sol.read_text())["status"] == "Optimal"
    r = subprocess.run([cli_bin, "solve", str(d / "r4.mps"), "--eps", "1e-12", "--iter-limit", "64"],
                       capture_output=True, text=True)
    assert r.returncode == 2 and "status=IterLimit" in r.stdout


@pytest.mark.gpu
def test_cpp_cli_device_and_shards(tmp_path):
    """Harness extension: `bench --gpus N --shards P` and
    `solve --device D --shards P` run the suite / solve with K split into P
    blocks (in-process shard mode) on the chosen devices; same statuses and
    objectives (1e-6) as the unsharded run, records in name order."""
    import subprocess
    cli_bin = _cpp_cli()
    d = tmp_path / "suite"
    d.mkdir()
    for seed in (4, 5, 6):
        rpdlp.WriteMpsFile(rpdlp.GenRandomLp(30, 40, 0.2, seed), d / f"r{seed}.mps")
    reps = {}
    for shards in (1, 3):
        rep = tmp_path / f"rep{shards}.json"
        r = subprocess.run([cli_bin, "bench", str(d), "--eps", "1e-6", "--gpus", "1", "--shards", str(shards),
                            "--report", str(rep)], capture_output=True, text=True)
        assert r.returncode == 0 and "solved=3/3" in r.stdout, r.stdout + r.stderr
        reps[shards] = json.loads(rep.read_text())
    a, b = reps[1]["records"], reps[3]["records"]
    assert [x["instance"] for x in a] == [x["instance"] for x in b] == ["r4.mps", "r5.mps", "r6.mps"]
    for x, y in zip(a, b):
        assert x["status"] == y["status"] == "Optimal"
        po, qo = x["residuals"]["primal_obj"], y["residuals"]["primal_obj"]
        assert abs(po - qo) <= 1e-6 * (1 + abs(po))
    r = subprocess.run([cli_bin, "solve", str(d / "r4.mps"), "--eps", "1e-6", "--device", "0", "--shards", "2"],
                       capture_output=True, text=True)
    assert r.returncode == 0 and "status=Optimal" in r.stdout, r.stdout + r.stderr
    r = subprocess.run([cli_bin, "solve", str(d / "r4.mps"), "--shards", "0"], capture_output=True, text=True)
    assert r.returncode != 0

"""CLI (reference SPEC.md:531-594): commands, reproducibility and exit codes 0/1/2/3."""
import json

from paper_2503_13737_b200 import cli, workload


def test_gen_reproducible_and_summary(tmp_path, capsys):
    a, b = tmp_path / "a.jsonl", tmp_path / "b.jsonl"
    assert cli.main(["gen", "--out", str(a), "--requests", "200", "--seed", "7"]) == 0
    summary = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert cli.main(["gen", "--out", str(b), "--requests", "200", "--seed", "7"]) == 0
    assert a.read_text() == b.read_text() and len(a.read_text().splitlines()) == 200
    assert summary["count"] == 200 if "count" in summary else True


def test_gen_invalid_rate_is_config_error(tmp_path):
    assert cli.main(["gen", "--out", str(tmp_path / "x.jsonl"), "--rate", "0"]) == 1


def test_run_two_policies_deterministic_then_compare(tmp_path, capsys):
    tr = tmp_path / "t.jsonl"
    assert cli.main(["gen", "--out", str(tr), "--requests", "40", "--rate", "4", "--long-fraction", "0"]) == 0
    outs = []
    for d in ("r1", "r2"):
        rc = cli.main(["run", "--trace", str(tr), "--policy", "paged_fcfs", "--policy", "accelgen",
                       "--horizon", "30", "--out", str(tmp_path / d)])
        assert rc == 0
        outs.append((tmp_path / d / "report.csv").read_text())
    assert outs[0] == outs[1]                       # same cfg twice -> identical CSVs
    assert len(outs[0].strip().splitlines()) == 3   # header + 2 policies
    capsys.readouterr()
    rc = cli.main(["compare", str(tmp_path / "r1" / "report_accelgen.json"),
                   str(tmp_path / "r1" / "report_paged_fcfs.json"), "--baseline", "paged_fcfs"])
    assert rc == 0
    table = json.loads(capsys.readouterr().out)
    assert set(table["ratios"]) == {"accelgen"}
    rc = cli.main(["compare", str(tmp_path / "r1" / "report_accelgen.json"),
                   str(tmp_path / "r2" / "report_accelgen.json"), "--baseline", "accelgen"])
    assert rc == 0  # identical reports -> no other policy, empty ratio table


def test_run_missing_profile_is_io_error(tmp_path):
    assert cli.main(["run", "--policy", "accelgen", "--profile", str(tmp_path / "nope.json"),
                     "--out", str(tmp_path / "o")]) == 2


def test_calibrate_idempotent_and_derive(tmp_path):
    full = tmp_path / "p.json"
    full.write_text(json.dumps({"hidden_size": 5120, "num_layers": 40, "pivot_forward_size": 768,
                                "pivot_time_s": 0.156}))
    out = tmp_path / "q.json"
    assert cli.main(["calibrate", "--profile", str(full), "--out", str(out)]) == 0
    assert json.loads(out.read_text())["pivot_forward_size"] == 768
    part = tmp_path / "part.json"
    part.write_text(json.dumps({"hidden_size": 5120, "num_layers": 40}))
    assert cli.main(["calibrate", "--profile", str(part), "--out", str(out)]) == 1  # X absent and S_pf absent
    gpu = tmp_path / "gpu.json"
    gpu.write_text(json.dumps({"peak_flops": 126.96e12}))
    assert cli.main(["calibrate", "--profile", str(part), "--gpu", str(gpu), "--out", str(out)]) == 0
    assert json.loads(out.read_text())["pivot_forward_size"] > 0


import pytest  # noqa: E402


@pytest.mark.gpu
def test_run_on_the_b200_executor(tmp_path):
    """`run --executor cuda`: the engine drives the OPT-13B forward on the GPU (device clock)."""
    tr = tmp_path / "t.jsonl"
    assert cli.main(["gen", "--out", str(tr), "--requests", "30", "--rate", "8", "--long-fraction", "0"]) == 0
    rc = cli.main(["run", "--trace", str(tr), "--policy", "accelgen", "--executor", "cuda", "--horizon", "2",
                   "--profile", "profiles/opt13b_b200_tp1.json", "--out", str(tmp_path / "o")])
    assert rc == 0
    rows = (tmp_path / "o" / "report.csv").read_text().strip().splitlines()
    assert len(rows) == 2 and rows[1].startswith("accelgen,")
    rep = json.loads((tmp_path / "o" / "report_accelgen.json").read_text())
    assert rep["tokens_per_s"] > 0

"""Command line: exit codes without a GPU, a run with one (reference tests/test_cli.py)."""
import json

import pytest

from paper_1403_7209_b200 import apps, cli, meshio


def test_bad_flags_exit_64(capsys):
    assert cli.main(["bench", "nope"]) == cli.EX_USAGE
    assert cli.main(["bench", "diffusion", "--backend", "threads"]) == cli.EX_USAGE
    assert cli.main([]) == cli.EX_USAGE


def test_mesh_errors_exit_65(tmp_path, capsys):
    bad = tmp_path / "bad.txt"
    bad.write_text("sets 1\nn x\n")
    assert cli.main(["bench", "diffusion", "--mesh", str(bad)]) == cli.EX_DATAERR
    assert "bad mesh file" in capsys.readouterr().err
    assert cli.main(["bench", "diffusion", "--mesh", str(tmp_path / "missing")]) == cli.EX_DATAERR
    # a mesh without the sets the app needs
    plain = tmp_path / "plain.txt"
    plain.write_text("sets 1\nn 2\nmaps 0\ndats 0\n")
    assert cli.main(["bench", "cell-area", "--mesh", str(plain)]) == cli.EX_DATAERR


@pytest.mark.gpu
def test_cli_runs_and_reports(tmp_path, capsys):
    path = tmp_path / "m.txt"
    meshio.dump_mesh(apps.gen_mesh(12), path)
    rep = tmp_path / "r.json"
    assert cli.main(["bench", "diffusion", "--mesh", str(path), "--steps", "3",
                     "--renumber", "on", "--report", str(rep)]) == 0
    doc = json.loads(rep.read_text())
    assert doc["config"]["backend"] == "cuda"
    assert len(doc["globals"]["residuals"]) == 3
    assert cli.main(["bench", "proxy", "--n", "10", "--steps", "1", "--tune", "schedule",
                     "--tune-table", str(tmp_path / "t.json"),
                     "--report", str(tmp_path / "r.csv")]) == 0
    assert (tmp_path / "t.json").exists()
    assert cli.main(["bench", "cell-area", "--report", str(tmp_path / "no" / "r.json")]) == cli.EX_IOERR

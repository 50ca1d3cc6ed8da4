"""bench-cli: CPU-side checks, and small device runs of every command."""
import csv
import os

import pytest

from paper_2209_05069_b200 import cli, io


def test_missing_pocket_file_exit_code(tmp_path, capsys):
    lig = tmp_path / "l.ligq"
    io.write_ligand_file(str(lig), io.generate_dataset(6, 1, 2, seed=1))
    rc = cli.console_main(["dock", "--ligands", str(lig), "--pocket", str(tmp_path / "nope.pock"),
                           "--out", str(tmp_path / "o")])
    assert rc == 2
    assert "nope.pock" in capsys.readouterr().err


def test_parser_flags():
    a = cli.build_parser().parse_args(["heatmap", "--engine", "latency", "--workers", "3", "--restarts", "4",
                                       "--top-k", "2", "--early-exit", "off", "--capacity-override", "0=64"])
    assert (a.engine, a.workers, a.restarts, a.top_k, a.early_exit) == ("latency", 3, 4, 2, "off")
    assert cli._caps(a) == {0: 64}


@pytest.mark.gpu
def test_heatmap_rows_and_determinism(tmp_path):
    args = ["heatmap", "--heavy", "8,12", "--frags", "1,4", "--count", "40", "--workers", "4"]
    assert cli.console_main(args + ["--out", str(tmp_path / "a")]) == 0
    rows = list(csv.reader(open(tmp_path / "a" / "heatmap.csv")))
    assert rows[0] == ["heavy_atoms", "fragments", "latency_tput", "batched_tput", "speedup"]
    assert [(r[0], r[1]) for r in rows[1:]] == [("8", "1"), ("8", "4"), ("12", "1"), ("12", "4")]
    assert all(float(r[4]) > 0 for r in rows[1:])


@pytest.mark.gpu
def test_scaling_and_ablation_and_dock(tmp_path, synth_pocket):
    assert cli.console_main(["scaling", "--max-size", "100", "--workers", "4", "--out", str(tmp_path / "s")]) == 0
    rows = list(csv.reader(open(tmp_path / "s" / "scaling.csv")))
    assert len(rows) - 1 == 2 * 2 * 2                                # |ladder| x 2 modes x 2 engines
    size10 = [r for r in rows[1:] if r[0] == "10" and r[2] == "batched"]
    assert all(float(r[5]) < 0.05 for r in size10)                   # SPEC.md:510, acceptance 8
    assert cli.console_main(["ablate-early-exit", "--heavy", "12", "--frags", "4", "--count", "30", "--workers", "4",
                             "--out", str(tmp_path / "e")]) == 0
    lig, poc = tmp_path / "l.ligq", tmp_path / "p.pock"
    io.write_ligand_file(str(lig), io.generate_dataset(10, 2, 20, seed=3))
    io.write_pocket_file(str(poc), synth_pocket)
    assert cli.console_main(["dock", "--ligands", str(lig), "--pocket", str(poc), "--out", str(tmp_path / "d")]) == 0
    out = list(csv.reader(open(tmp_path / "d" / "results.csv")))
    assert out[0] == ["ligand_id", "geom_score", "chem_score", "valid"] and len(out) == 21


@pytest.mark.gpu
def test_dock_exits_nonzero_on_fatal_config(tmp_path):
    """An engine's fatal error (a configuration the device rejects) gives a non-zero exit status."""
    from paper_2209_05069_b200 import io
    lig, pock = tmp_path / "l.ligq", tmp_path / "p.pock"
    io.write_ligand_file(str(lig), io.generate_dataset(12, 2, 3, seed=1))
    io.write_pocket_file(str(pock), io.synthetic_pocket())
    args = ["dock", "--ligands", str(lig), "--pocket", str(pock), "--workers", "2", "--out", str(tmp_path / "o")]
    assert cli.console_main(args) == 0
    from paper_2209_05069_b200 import model
    orig = cli._cfg
    cli._cfg = lambda a: model.DockConfig(alignment_step_deg=1)
    try:
        assert cli.console_main(args) == 1
    finally:
        cli._cfg = orig

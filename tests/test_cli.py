"""Experiment drivers (paper_2101_08053_b200.cli) with the reference CLI's
command line and CSV formats (src/cli.py; the reference's own checks in
pkg/tests/test_cli.py are the model).  Configuration handling runs on CPU;
the commands form matrices on the GPU."""

import csv
import json

import numpy as np
import pytest


def read_csv(path):
    with open(path) as fh:
        rows = list(csv.reader(fh))
    return rows[0], rows[1:]


def test_run_config_validation_and_strategies():
    from paper_2101_08053_b200.cli import RunConfig
    for bad in (dict(case="sphere"), dict(degrees=[0]), dict(degrees=[7]), dict(meshes=[])):
        with pytest.raises(ValueError):
            RunConfig(**bad)
    cfg = RunConfig()
    assert cfg.strategies("mass") == ("reference", "wq", "hybrid", "dwq")
    assert cfg.strategies("converge") == ("reference", "hybrid", "dwq")
    assert RunConfig(strategy="hybrid").strategies("time") == ("hybrid",)
    with pytest.raises(ValueError):
        RunConfig(strategy="gauss").strategies("mass")


def test_argument_parsing_and_defaults(tmp_path):
    from paper_2101_08053_b200.cli import _config_from_args, _parse_int_list, _parser
    assert _parse_int_list("1..4") == [1, 2, 3, 4] and _parse_int_list("2,4,6") == [2, 4, 6]
    c = _config_from_args(_parser().parse_args(["mass"]))
    assert c.meshes == [10] and c.degrees == [1, 2, 3, 4, 5, 6] and c.case == "line"
    c = _config_from_args(_parser().parse_args(["time", "--case", "corner"]))
    assert c.degrees == [2, 3, 4, 5, 6] and c.meshes == [5, 10, 20, 40]
    knots = {"degree": 2, "knots": [0, 0, 0, 0.2, 0.55, 0.55, 0.8, 1, 1, 1]}
    (tmp_path / "run.json").write_text(json.dumps({"case": "circle", "degrees": "2..3", "knots1": knots,
                                                   "out": str(tmp_path)}))
    c = _config_from_args(_parser().parse_args(["converge", "--config", str(tmp_path / "run.json"),
                                                "--meshes", "4,8"]))
    assert c.case == "circle" and c.degrees == [2, 3] and c.meshes == [4, 8]
    assert c.knots1.degree == 2 and c.knots2 is None and c.out == tmp_path


@pytest.mark.gpu
def test_mass_table_contents(tmp_path):
    from paper_2101_08053_b200.cli import main
    assert main(["mass", "--case", "line", "--degrees", "1..2", "--meshes", "8", "--out", str(tmp_path)]) == 0
    header, rows = read_csv(tmp_path / "mass_line_n8.csv")
    assert header == ["degree", "hybrid_gauss", "disc_weighted_quadrature", "weighted_quadrature",
                      "hybrid_rel", "dwq_rel", "wq_rel", "reference_frobenius"]
    for row in rows:
        assert float(row[4]) <= 1e-12 and float(row[5]) <= 1e-12
        assert 1e-6 <= float(row[3]) <= 1e-2        # naive WQ: the paper's failure band


@pytest.mark.gpu
def test_mass_dumps_and_determinism(tmp_path):
    from paper_2101_08053_b200.cli import main
    main(["mass", "--case", "line", "--degrees", "2", "--meshes", "6", "--out", str(tmp_path),
          "--dump-rules", str(tmp_path / "rules.json"), "--dump-cutcells", str(tmp_path / "cut.csv")])
    rules = json.loads((tmp_path / "rules.json").read_text())
    assert {r["direction"] for r in rules} == {0, 1}
    assert all(r["rows"] and r["points"] for r in rules)
    header, rows = read_csv(tmp_path / "cut.csv")
    assert header == ["u1", "u2", "weight"] and all(float(r[2]) > 0 for r in rows)
    args = ["mass", "--case", "circle", "--degrees", "1,2", "--meshes", "6"]
    main(args + ["--out", str(tmp_path / "a")])
    main(args + ["--out", str(tmp_path / "b")])
    assert (tmp_path / "a" / "mass_circle_n6.csv").read_bytes() == (tmp_path / "b" / "mass_circle_n6.csv").read_bytes()


@pytest.mark.gpu
def test_converge_records_and_summary(tmp_path):
    from paper_2101_08053_b200.cli import main
    main(["converge", "--case", "line", "--degrees", "1", "--meshes", "5,10,20", "--out", str(tmp_path)])
    header, rows = read_csv(tmp_path / "convergence_line.csv")
    assert header == ["case", "strategy", "p", "h", "dofs", "l2_rel", "rate"]
    assert {r[1] for r in rows} == {"reference", "hybrid", "dwq"}
    sheader, srows = read_csv(tmp_path / "convergence_line_summary.csv")
    assert sheader == ["case", "strategy", "p", "observed_rate", "rate_check", "ref_agreement"]
    for row in srows:
        assert row[4] == "PASS" and float(row[5]) <= 1e-10


@pytest.mark.gpu
def test_converge_matches_oracle_errors(tmp_path):
    """The errors of the study agree with the oracle's (1e-10 absolute)."""
    from oracle import configs as OC, project as OP, assemble as OA
    from paper_2101_08053_b200.cli import main
    main(["converge", "--case", "circle", "--degrees", "2", "--meshes", "6,12", "--strategy", "hybrid",
          "--out", str(tmp_path)])
    _, rows = read_csv(tmp_path / "convergence_circle.csv")
    for row in rows:
        nel = round(1.0 / float(row[3]))
        cfg = OC.build_space([OC.case_curve("circle")], nel, 2)
        M = OA.assemble_mass(cfg, strategy="hybrid")
        b = OP.assemble_rhs(OP.default_target, cfg)
        x = OP.solve_spd(M.data, b)
        e = OP.l2_error(x, OP.default_target, cfg)
        assert abs(float(row[5]) - e) <= 1e-10


@pytest.mark.gpu
def test_time_columns_and_counts(tmp_path):
    from oracle import assemble as OA, configs as OC
    from paper_2101_08053_b200.cli import main
    main(["time", "--case", "line", "--degrees", "2", "--meshes", "5", "--out", str(tmp_path)])
    header, rows = read_csv(tmp_path / "timings_line_n5.csv")
    assert header == ["strategy", "case", "p", "h", "t_weights", "t_interior", "t_cutRegular", "t_cutElements",
                      "t_total", "n_wq_points", "n_gauss_elements", "n_cutcell_points"]
    assert [r[0] for r in rows] == ["reference", "hybrid", "dwq"]
    cfg = OC.build_space([OC.case_curve("line")], 5, 2)
    for r in rows:
        assert float(r[8]) > 0
        _, rep = OA.form_with_timings(r[0], cfg)
        assert (int(r[9]), int(r[10]), int(r[11])) == (rep.n_wq_points, rep.n_gauss_elements,
                                                        rep.n_cutcell_points), r[0]

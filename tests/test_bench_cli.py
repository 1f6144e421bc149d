"""The GPU ntd-bench keeps the reference CLI's schema and exit codes
(/root/reference/pkg/tests/test_bench_cli.py): parser defaults, validation,
report renderings, exit codes (CPU); real runs on the device (gpu)."""

import json

import pytest

from paper_1909_09771_b200 import bench_cli
from paper_1909_09771_b200.banded_core import FactorizationError
from paper_1909_09771_b200.bench_cli import (CSV_HEADER, BenchConfig, BenchReport, main, make_parser,
                                             run_benchmark)


def tiny_config(**kw):
    cfg = BenchConfig(matrix_type=3, n=6, tol=1e-6, max_iters=100)
    for key, val in kw.items():
        setattr(cfg, key, val)
    return cfg


def fake_report(**kw):
    d = dict(matrix_type=3, rows=216, tol=1e-6, workers=1, precond="ntd+ilu0", assembly_seconds=0.01,
             setup_seconds=0.25, solve_seconds=0.5, iterations=3, converged=True, final_relres=4e-7,
             residual_history=[1e-2, 1e-4, 4e-7])
    d.update(kw)
    return BenchReport(**d)


def test_parser_defaults():
    args = make_parser().parse_args([])
    assert (args.matrix_type, args.n, args.tol) == (3, 50, 1e-7)
    assert (args.max_iters, args.workers) == (200, 1)
    assert (args.rhs_mode, args.precond, args.output_format) == ("ones", "ntd+ilu0", "table")
    assert args.dump_matrix is None and args.speedup is False


def test_config_validation():
    for kw in (dict(matrix_type=4), dict(n=0), dict(tol=-1.0), dict(max_iters=0), dict(workers=3),
               dict(rhs_mode="junk"), dict(precond="amg"), dict(output_format="xml")):
        with pytest.raises(ValueError):
            tiny_config(**kw).validate()
    tiny_config().validate()


def test_report_renderings():
    r = fake_report()
    doc = json.loads(r.to_json())
    assert doc["overall_seconds"] == pytest.approx(0.75)
    assert set(doc) == {"matrix_type", "rows", "tol", "workers", "precond", "assembly_seconds", "setup_seconds",
                        "solve_seconds", "iterations", "converged", "final_relres", "residual_history",
                        "overall_seconds"}
    head, row = r.to_csv().splitlines()
    assert head == CSV_HEADER and row.split(",")[:3] == ["3", "216", "1e-06"] and row.split(",")[6] == "3"
    table = r.to_table()
    assert "iterations      : 3 (converged)" in table
    assert "NOT CONVERGED" in fake_report(converged=False).to_table()
    assert r.rendered("json") == r.to_json() and r.rendered("csv") == r.to_csv()


def test_exit_codes_without_a_solve(monkeypatch, capsys):
    assert main(["--n", "0"]) == 2  # validation error
    monkeypatch.setattr(bench_cli, "run_benchmark",
                        lambda cfg: (_ for _ in ()).throw(FactorizationError("zero pivot at row 3")))
    assert main(["--n", "4"]) == 4  # numerical failure
    monkeypatch.setattr(bench_cli, "run_benchmark", lambda cfg: fake_report(converged=False))
    assert main(["--n", "4", "--format", "csv"]) == 3  # iteration limit
    assert capsys.readouterr().out.startswith(CSV_HEADER)


@pytest.mark.gpu
@pytest.mark.parametrize("precond", bench_cli.PRECOND_CHOICES)
@pytest.mark.parametrize("rhs_mode", ("ones", "manufactured"))
def test_gpu_run_schema(precond, rhs_mode):
    report = run_benchmark(tiny_config(precond=precond, rhs_mode=rhs_mode))
    doc = json.loads(report.to_json())
    assert doc["converged"] and doc["rows"] == 216 and doc["final_relres"] < 1e-6
    assert doc["iterations"] == len(doc["residual_history"])


@pytest.mark.gpu
def test_gpu_main_exit_codes(capsys, tmp_path):
    assert main(["--n", "6", "--tol", "1e-6", "--format", "json"]) == 0
    assert json.loads(capsys.readouterr().out)["converged"]
    assert main(["--n", "12", "--precond", "none", "--max-iters", "2", "--tol", "1e-12"]) == 3
    path = tmp_path / "a.mtx"
    assert main(["--n", "3", "--dump-matrix", str(path)]) == 0 and path.exists()

"""Harness / CLI, modelled on the reference's
test_bench.py: configuration validation, sweeps, CSV round trip (both the
reference's 12-column layout and the extended one), CLI exit codes through
click's CliRunner (CPU); one small device sweep (GPU)."""

import numpy as np
import pytest

from paper_2403_16013_b200 import harness as hb


def test_config_validation_and_sweep():
    assert hb.BenchConfig(n=100).validate().sweep() == [32, 64, 96]
    assert hb.BenchConfig(n=20).validate().sweep() == [20]
    assert hb.BenchConfig(n=64, algorithm="normal").validate().sweep() == [64]
    assert hb.BenchConfig(n=64, k_values=[8, 16]).validate().sweep() == [8, 16]
    for bad in (dict(n=0), dict(reps=0), dict(algorithm="x"), dict(precision="hd"),
                dict(n=8, k_values=[9]), dict(threads=[0]), dict(kernel="strassen"),
                dict(splits=0)):
        with pytest.raises(ValueError):
            hb.BenchConfig(**bad).validate()
    assert hb.BenchConfig(precision="td").effective_splits(3) == 8


def _rec(**kw):
    base = dict(precision="dd", algorithm="blocked", method="3m", kernel="b200", n=64, K=32,
                splits=6, threads=1, rep_median_seconds=0.125, max_relerr="1e-30", seed=1,
                status="ok")
    base.update(kw)
    return hb.BenchRecord(**base)


@pytest.mark.parametrize("extended", [False, True])
def test_csv_round_trip(tmp_path, extended):
    recs = [_rec(), _rec(K=64, status="singular", gflops_conv=12.5, fp64_pct=80.0,
                         pivots_equal=False, bwd_err=3e-31)]
    p = tmp_path / "out.csv"
    hb.emit_csv(recs, str(p), extended=extended)
    back = hb.read_csv(str(p))
    assert [r.row() for r in back] == [r.row() for r in recs]
    if extended:
        assert back[1].gflops_conv == 12.5 and back[1].pivots_equal is False
        assert back[1].bwd_err == 3e-31
    head = open(p).readline().strip().split(",")
    assert head[:12] == hb.CSV_COLUMNS


def test_csv_rejects_bad_header(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("a,b\n1,2\n")
    with pytest.raises(ValueError):
        hb.read_csv(str(p))


def test_factor_op_model():
    # K = n: a single panel, no TRSM / GEMM: n (n-1)/2 * n-ish panel updates
    ops = hb._factor_ops(4, 4, 2, "3m", True)
    assert ops == (3 * 3 + 2 * 2 + 1 * 1) * 173   # sum_j (rows below j) (columns right of j)
    # n = 8, K = 4: panels 38 + 14 updates, TRSM 4 * 6, GEMM 4 * 4 * 4 complex MACs
    assert hb._factor_ops(8, 4, 2, "3m", False) == (38 + 14 + 24) * 173 + 64 * 93


def test_cli_usage_errors():
    from click.testing import CliRunner

    from paper_2403_16013_b200.cli import cli

    r = CliRunner().invoke(cli, ["bench", "--n", "0"])
    assert r.exit_code != 0
    r = CliRunner().invoke(cli, ["bench", "--k-sweep", "1:2:3:4"])
    assert r.exit_code != 0
    r = CliRunner().invoke(cli, ["bench", "--gpus", "2"])
    assert r.exit_code != 0
    r = CliRunner().invoke(cli, ["--help"])
    assert r.exit_code == 0 and "matmul-bench" in r.output


@pytest.mark.gpu
def test_gpu_cli_bench_and_verify(tmp_path):
    from click.testing import CliRunner

    from paper_2403_16013_b200.cli import cli

    out = tmp_path / "b.csv"
    r = CliRunner().invoke(cli, ["bench", "--n", "64", "--k-sweep", "32:64:32", "--reps", "2",
                                 "--csv", str(out), "--verify", "--strict"])
    assert r.exit_code == 0, r.output
    recs = hb.read_csv(str(out))
    assert [x.K for x in recs] == [32, 64]
    assert all(x.status == "ok" and x.pivots_equal and x.gflops_conv > 0 for x in recs)
    assert all(float(x.max_relerr) < 1e-25 and x.bwd_err < 1e-28 for x in recs)
    r = CliRunner().invoke(cli, ["matmul-bench", "--n", "48", "--kernel", "ozaki", "--check",
                                 "--strict"])
    assert r.exit_code == 0, r.output
    for suite in ("matmul", "lu"):
        r = CliRunner().invoke(cli, ["verify", "--suite", suite])
        assert r.exit_code == 0 and "FAIL" not in r.output, r.output

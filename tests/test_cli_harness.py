"""The B200 harness/CLI against the reference CLI's own output: under
--deterministic the CSV holds only configuration and audited counters, so it
must be byte-identical to the reference's (tests/golden/cli.json, produced by
running the reference CLI)."""

import contextlib
import io
import json

import pytest

from conftest import GOLDEN

CASES = json.loads((GOLDEN / "cli.json").read_text())


def _run(argv):
    from paper_2501_03121_b200.cli import main

    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = main(argv)
    return rc, out.getvalue(), err.getvalue()


@pytest.mark.parametrize("case", [c for c in CASES if c["rc"] != 0], ids=lambda c: " ".join(c["argv"][:3]))
def test_configuration_errors_exit_2_without_a_gpu(case):
    rc, out, err = _run(case["argv"])
    assert rc == case["rc"] == 2 and out == case["stdout"] and "configuration error" in err


COST_CASES = json.loads((GOLDEN / "cli_cost.json").read_text())


@pytest.mark.parametrize("case", COST_CASES, ids=lambda c: " ".join(c["argv"][1:]))
def test_cost_subcommand_byte_identical_to_reference(case):
    """`cost` evaluates the closed forms (no GPU): same CSV bytes and exit
    codes as the reference CLI (cli.py:147-156)."""
    rc, out, err = _run(case["argv"])
    assert rc == case["rc"] and out == case["stdout"], err


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in CASES if c["rc"] == 0], ids=lambda c: " ".join(c["argv"][:5]))
def test_deterministic_csv_byte_identical_to_reference(tv, case):
    rc, out, err = _run(case["argv"])
    assert rc == 0, err
    assert out == case["stdout"]


@pytest.mark.gpu
def test_timed_run_and_grid(tv):
    from paper_2501_03121_b200 import harness as H

    res = H.run_bench(H.BenchConfig("tvc", H.parse_dims("64^3"), k=1, iters=3, peak=6.4e12))
    assert res.iterations == 3 and res.touched_pred == res.touched_meas and res.bytes_s > 0
    assert res.norm_bw_pct is not None
    results, stats = H.sweep_grid(H.BenchConfig("tvc", H.parse_dims("32^3"), iters=2))
    assert stats.runs == 3 and stats.mean_bytes_s > 0
    buf = io.StringIO()
    H.emit_csv(results, buf)
    assert buf.getvalue().count("\n") == 4
    tri = H.stream_triad(1 << 20, iters=2)
    assert tri.touched_meas == 3 << 20

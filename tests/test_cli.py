"""CPU tests of the CLI front end (reference formats, tools/commands.cpp)."""
import os

import numpy as np
import pytest

from oracle_bindings import Oracle
from paper_1604_05140_b200 import cli
from conftest import gpu_available


def test_coefficient_stream_matches_reference_draw():
    """CoefficientStream (commands.cpp:73-88) == the acceptance suite's draw
    (acceptance_main.cpp:50-63), as restated by the oracle's mt19937_64."""
    for B, seed in ((2, 0), (8, 1042), (16, 7)):
        a = cli.CoefficientStream(seed).next(B)
        assert np.array_equal(a, Oracle.random_coefficients(B, seed))
    s = cli.CoefficientStream(5)
    first, second = s.next(4), s.next(4)
    both = cli.CoefficientStream(5).next(8)  # stream continues across calls
    assert not np.array_equal(first, second)


def test_csv_roundtrip_format(tmp_path):
    path = tmp_path / "r.csv"
    recs = [dict(B=16, variant="fast", reps=10, mean_time_s=1.25e-4, mean_max_abs_err=3.1e-15,
                 mean_max_rel_err=7.0e-14)]
    cli.append_csv(str(path), recs)
    cli.append_csv(str(path), recs)
    lines = path.read_text().splitlines()
    assert lines[0] == "B,variant,reps,mean_time_s,mean_max_abs_err,mean_max_rel_err"
    assert lines[1] == "16,fast,10,0.000125,%.17g,%.17g" % (3.1e-15, 7.0e-14)  # printf("%.17g")
    assert len(lines) == 3
    back = cli.read_csv(str(path))
    assert back[0] == recs[0] and len(back) == 2
    assert cli.record_line(recs[0]) == "  16  fast         10      0.000125   3.100000e-15   7.000000e-14"


def test_usage_errors_exit_2():
    assert cli.main(["roundtrip"]) == 2
    assert cli.main(["transform", "--direction", "sideways", "--bandlimit", "2", "--in", "x", "--out", "y"]) == 2
    assert cli.main([]) == 2


@pytest.mark.skipif(gpu_available(), reason="checks the no-device path")
def test_runtime_errors_exit_1(tmp_path, capsys):
    assert cli.main(["roundtrip", "--bandlimit", "4", "--repetitions", "1"]) == 1
    assert "error:" in capsys.readouterr().err
    bad = tmp_path / "in.bin"
    bad.write_bytes(b"\0" * 48)
    assert cli.main(["transform", "--direction", "fwd", "--bandlimit", "2", "--in", str(bad),
                     "--out", str(tmp_path / "o.bin")]) == 1

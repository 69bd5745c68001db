"""PGM frame IO and the benchmark CSV (SURVEY next-3) against the REAL
reference's behaviour (tests/golden/io/, made by make_golden_io.py):
decoded rasters, PgmError messages and byte offsets, written bytes, CSV text."""

import json
import os

import numpy as np
import pytest

from paper_1609_04567_b200.bench import BenchRow, RunSpec, emit_csv
from paper_1609_04567_b200.grid import Grid, GridError
from paper_1609_04567_b200.pgm import PgmError, read_pgm, write_pgm

IO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")
MAN = json.load(open(os.path.join(IO, "manifest.json")))


@pytest.mark.parametrize("name", sorted(MAN["read"]))
def test_read_matches_reference(name):
    g = read_pgm(os.path.join(IO, name))
    want = MAN["read"][name]
    assert list(g.dims) == want["dims"]
    data = g.data
    assert sum(data) == want["sum"] and data[:8] == want["first"] and data[-8:] == want["last"]
    assert all(type(v) is int for v in data[:8])


def test_p2_and_p5_agree():
    a = read_pgm(os.path.join(IO, "sample_p2.pgm")).to_array()
    b = read_pgm(os.path.join(IO, "sample_p5.pgm")).to_array()
    assert np.array_equal(a, b)


@pytest.mark.parametrize("name", sorted(MAN["errors"]))
def test_errors_match_reference(name):
    want = MAN["errors"][name]
    with pytest.raises(PgmError) as ei:
        read_pgm(os.path.join(IO, name))
    assert str(ei.value) == want["message"]
    assert ei.value.offset == want["offset"]
    assert isinstance(ei.value, GridError)


def test_writes_are_byte_identical(tmp_path):
    img = read_pgm(os.path.join(IO, "sample_p5.pgm"))
    a = img.to_array().astype(np.int64)
    for binary, name in ((True, "write_p5.pgm"), (False, "write_p2.pgm")):
        p = tmp_path / name
        write_pgm(p, Grid.from_array(a), binary=binary)
        assert p.read_bytes() == open(os.path.join(IO, name), "rb").read()
    p = tmp_path / "m.pgm"
    write_pgm(p, Grid.from_array(a % 101), binary=False, maxval=100)
    assert p.read_bytes() == open(os.path.join(IO, "write_p2_max100.pgm"), "rb").read()
    # floats that are whole numbers are fine, as in the reference
    write_pgm(p, Grid.from_array(a.astype(np.float64)))
    assert p.read_bytes() == open(os.path.join(IO, "write_p5.pgm"), "rb").read()


@pytest.mark.parametrize("rows,tag", [([[1.5, 2.0]], "frac"), ([[1, 300]], "range")])
def test_write_errors_match_reference(tmp_path, rows, tag):
    with pytest.raises(GridError) as ei:
        write_pgm(tmp_path / "x.pgm", Grid.from_rows(rows))
    assert str(ei.value) == MAN["write"]["err_" + tag]


def test_csv_text_matches_reference():
    rows = [BenchRow("sobel", "b.pgm", 1, 1, "1:1", 42, 1, 12.3456789, 1, 0, 1, 926609350),
            BenchRow("helmholtz", "unit-64x64", 4, 1, "1:n", 42, 36, 0.5, 4, 384, 4, 1.0187e-05),
            BenchRow("gol", "soup,\"q\"", 2, 3, "1:n", 7, 100, 1e-7, 2, 25600, 2, 510.0)]
    assert emit_csv(rows) == MAN["csv"]


def test_runspec_validation():
    with pytest.raises(GridError):
        RunSpec(app="", input_id="x")
    with pytest.raises(GridError):
        RunSpec(app="a", input_id="x", mode="1:n", partitions=1)
    assert RunSpec(app="a", input_id="x", mode="1:n", partitions=2).mode.value == "1:n"

"""The command line front end (paper_1609_04567_b200.cli) against the REAL
reference's `stencilkit` command (tests/golden/io/manifest.json, made by
make_golden_io.py): same stdout (wall_ms masked), exit status, CSV rows and
byte-identical output PGMs, for gol / helmholtz / sobel / denoise (image and
frame stream) and a failing input."""

import contextlib
import io
import json
import os
import re
import shutil

import pytest

from paper_1609_04567_b200 import cli

pytestmark = pytest.mark.gpu

IO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")
MAN = json.load(open(os.path.join(IO, "manifest.json")))
RUNS = sorted(k for k in MAN["cli"] if not k.startswith("csv:"))


@pytest.mark.parametrize("name", RUNS)
def test_cli_matches_reference(name, tmp_path):
    want = MAN["cli"][name]
    for f in ("sample_p5.pgm", "p5_truncated.pgm"):
        shutil.copy(os.path.join(IO, f), tmp_path / f)
    argv = [a.replace("{out}", str(tmp_path)) for a in want["argv"]]
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = cli.main(argv)
    assert rc == want["rc"]
    assert re.sub(r"wall_ms=[0-9.]+", "wall_ms=*", out.getvalue()) == want["stdout"]
    assert err.getvalue().replace(str(tmp_path), "{out}") == want["stderr"]
    # output images: byte-identical
    for a in argv:
        if a.startswith(str(tmp_path)) and a.endswith(".pgm") and "sample" not in a \
                and "truncated" not in a:
            assert open(a, "rb").read() == open(os.path.join(IO, os.path.basename(a)), "rb").read()
    for d in ("frames", "masks"):
        if (tmp_path / d).exists():
            names = sorted(os.listdir(tmp_path / d))
            assert names == sorted(os.listdir(os.path.join(IO, d)))
            for n in names:
                assert (tmp_path / d / n).read_bytes() == open(os.path.join(IO, d, n), "rb").read()
    for a in argv:
        if a.endswith(".csv"):
            txt = open(a).read()
            masked = re.sub(r"(,)[0-9.e+-]+(,[0-9]+,[0-9]+,[0-9]+,[^,]*\r?\n)", r"\1*\2", txt)
            assert masked == MAN["cli"]["csv:" + os.path.basename(a)]

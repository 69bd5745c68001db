"""Golden fixtures for the formats either side of the stream (SURVEY next-3),
made with the REAL reference (build container only):

    python tests/golden/make_golden_io.py

* PGM: sample P2 / P5 files (comments, odd whitespace), what the reference's
  read_pgm returns for them, its PgmError message + offset for malformed
  variants, and the exact bytes its write_pgm produces;
* CSV: emit_csv text for a few rows;
* CLI: stdout (wall_ms masked), output PGM bytes and CSV rows of the
  reference's `stencilkit` command for small gol / helmholtz / sobel /
  denoise (image and frame stream) runs.

Everything lands in tests/golden/io/ (manifest.json + the files).
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import re
import shutil
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "io")

MALFORMED = {
    "bad_magic.pgm": b"P6\n2 2\n255\n\x00\x01\x02\x03",
    "bad_width.pgm": b"P2\n2x 2\n255\n1 2 3 4\n",
    "zero_dims.pgm": b"P2\n0 2\n255\n",
    "big_maxval.pgm": b"P2\n2 2\n65535\n1 2 3 4\n",
    "p2_value_range.pgm": b"P2\n2 2\n100\n1 2 300 4\n",
    "p2_bad_token.pgm": b"P2\n2 2\n255\n1 2 x3 4\n",
    "p2_short.pgm": b"P2\n3 2\n255\n1 2 3 4\n# end\n",
    "p5_no_ws.pgm": b"P5\n2 2\n255#c\n\x00\x01\x02\x03",
    "p5_truncated.pgm": b"P5\n4 4\n255\n\x00\x01\x02",
    "p5_over_maxval.pgm": b"P5\n3 1\n200\n\x05\xc9\x07",
    "header_eof.pgm": b"P2\n# only a comment\n 7 ",
}


def main():
    sys.path.insert(0, REF)
    from stencilkit import pgm as R
    from stencilkit import cli as RC
    from stencilkit.bench import BenchRow, emit_csv
    from stencilkit.grid import Grid

    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(OUT)
    man = {"read": {}, "errors": {}, "write": {}, "csv": None, "cli": {}}
    rng = np.random.default_rng(7)
    img = rng.integers(0, 256, (23, 31))
    # valid inputs
    p5 = b"P5\n# made by hand\n31 23\n255\n" + img.astype(np.uint8).tobytes()
    p2 = ("P2\n31 23 # dims\n255\n" + "\n".join(
        "  ".join(str(v) for v in row) + (" # row" if i % 5 == 0 else "")
        for i, row in enumerate(img)) + "\n").encode()
    for name, data in (("sample_p5.pgm", p5), ("sample_p2.pgm", p2), *MALFORMED.items()):
        with open(os.path.join(OUT, name), "wb") as fh:
            fh.write(data)
    for name in ("sample_p5.pgm", "sample_p2.pgm"):
        g = R.read_pgm(os.path.join(OUT, name))
        man["read"][name] = {"dims": list(g.dims), "sum": int(sum(g.data)),
                             "first": g.data[:8], "last": g.data[-8:]}
    for name in MALFORMED:
        try:
            R.read_pgm(os.path.join(OUT, name))
            man["errors"][name] = None
        except R.PgmError as e:
            man["errors"][name] = {"message": str(e), "offset": e.offset}
    # writes
    g = Grid.from_array(img)
    for binary in (True, False):
        path = os.path.join(OUT, f"write_{'p5' if binary else 'p2'}.pgm")
        R.write_pgm(path, g, binary=binary)
        man["write"][os.path.basename(path)] = True
    R.write_pgm(os.path.join(OUT, "write_p2_max100.pgm"),
                Grid.from_array(img % 101), binary=False, maxval=100)
    man["write"]["write_p2_max100.pgm"] = True
    for bad, tag in (([[1.5, 2.0]], "frac"), ([[1, 300]], "range")):
        try:
            R.write_pgm(os.path.join(OUT, "x.pgm"), Grid.from_rows(bad))
        except Exception as e:
            man["write"]["err_" + tag] = str(e)
    # csv
    rows = [BenchRow("sobel", "b.pgm", 1, 1, "1:1", 42, 1, 12.3456789, 1, 0, 1, 926609350),
            BenchRow("helmholtz", "unit-64x64", 4, 1, "1:n", 42, 36, 0.5, 4, 384, 4,
                     1.0187e-05),
            BenchRow("gol", "soup,\"q\"", 2, 3, "1:n", 7, 100, 1e-7, 2, 25600, 2, 510.0)]
    man["csv"] = emit_csv(rows)
    # the CLI
    runs = {
        "gol": ["gol", "--n", "40", "--m", "50", "-p", "2", "--mode", "1:n", "--seed", "3",
                "--max-iters", "12", "--out", "{out}/gol.pgm", "--csv", "{out}/gol.csv"],
        "helmholtz": ["helmholtz", "--n", "40", "--m", "33", "--tol", "1e-5", "--csv",
                      "{out}/helm.csv"],
        "sobel": ["sobel", "--in", "{out}/sample_p5.pgm", "--out", "{out}/sobel.pgm", "-p", "3",
                  "--mode", "1:n"],
        "denoise": ["denoise", "--n", "48", "--m", "40", "--noise-level", "0.3",
                    "--out", "{out}/denoise.pgm", "--csv", "{out}/denoise.csv"],
        "denoise_frames": ["denoise", "--frames", "3", "--n", "36", "--m", "44", "-w", "2",
                           "--out", "{out}/frames", "--noise-map-out", "{out}/masks"],
        "bad_input": ["sobel", "--in", "{out}/p5_truncated.pgm"],
    }
    for name, argv in runs.items():
        real = [a.replace("{out}", OUT) for a in argv]
        buf, ebuf = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(ebuf):
            rc = RC.main(real)
        man["cli"][name] = {"argv": argv, "rc": rc,
                            "stdout": re.sub(r"wall_ms=[0-9.]+", "wall_ms=*", buf.getvalue()),
                            "stderr": ebuf.getvalue().replace(OUT, "{out}")}
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".csv"):
            txt = open(os.path.join(OUT, f)).read()
            man["cli"]["csv:" + f] = re.sub(r"(,)[0-9.e+-]+(,[0-9]+,[0-9]+,[0-9]+,[^,]*\r?\n)",
                                            r"\1*\2", txt)
            os.remove(os.path.join(OUT, f))
    with open(os.path.join(OUT, "manifest.json"), "w") as fh:
        json.dump(man, fh, indent=1, sort_keys=True)
    print(json.dumps({k: (len(v) if isinstance(v, dict) else 1) for k, v in man.items()}))


if __name__ == "__main__":
    main()

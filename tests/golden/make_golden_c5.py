"""Golden fixtures for BASELINE C5 (streaming video denoise) frames 0..N-1.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden_c5.py [--frames 64] [--procs 8]

Frame i = salt_pepper(_synthetic_frame(1080, 1920, i), 0.1, seed=42+i)[0]
(cli.py:187-191, apps/denoise.py:295-304), detected with amf_detect and
restored with restore_regularize at P=1 by the REAL reference package
(stencilkit from /root/reference/pkg/src), one process per frame.  Records
per frame: flagged pixels, iterations, exhausted, final reduce, SHA-256 of
the fp64 output and of its rint/clip uint8 form (the CLI's PGM bytes,
cli.py:128-130).  Writes tests/golden/golden_c5.json.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def one(i):
    sys.path.insert(0, REF)
    from stencilkit.apps import amf_detect, restore_regularize, salt_pepper
    from stencilkit.cli import _synthetic_frame

    t0 = time.perf_counter()
    noisy = salt_pepper(_synthetic_frame(1080, 1920, i), 0.1, seed=42 + i)[0]
    mask = amf_detect(noisy)
    out, rep = restore_regularize(noisy, mask)
    a = np.asarray(out.to_array(), dtype=np.float64)
    m = mask.to_array()
    return i, dict(flagged=int(np.asarray(m).sum()), sha_mask=sha(np.asarray(m, np.uint8)),
                   iterations=rep.iterations, exhausted=rep.exhausted,
                   final_reduce=rep.final_reduce, sha=sha(a),
                   sha_u8=sha(np.clip(np.rint(a), 0, 255).astype(np.uint8)),
                   wall_s=time.perf_counter() - t0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=64)
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 8)
    ap.add_argument("--extend", action="store_true",
                    help="keep the frames already in golden_c5.json, compute the rest")
    args = ap.parse_args()
    out = {}
    path = os.path.join(HERE, "golden_c5.json")
    if args.extend and os.path.exists(path):
        out = dict(json.load(open(path))["frames"])
    todo = [i for i in range(args.frames) if str(i) not in out]
    with Pool(args.procs) as pool:
        for n, (i, rec) in enumerate(pool.imap_unordered(one, todo)):
            out[str(i)] = rec
            print(i, rec["iterations"], rec["flagged"], f"{rec['wall_s']:.1f}s", flush=True)
            if n % 64 == 63:  # checkpoint
                _write(path, out)
    _write(path, out)
    print("wrote", len(out), "frames")


def _write(path, out):
    meta = {"source": "reference stencilkit (P=1), tests/golden/make_golden_c5.py",
            "level": 0.1, "rows": 1080, "cols": 1920,
            "frames": {k: out[k] for k in sorted(out, key=int)}}
    with open(path + ".tmp", "w") as fh:
        json.dump(meta, fh, indent=1)
    os.replace(path + ".tmp", path)


if __name__ == "__main__":
    main()

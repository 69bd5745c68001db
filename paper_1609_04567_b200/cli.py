"""Command line front end (reference: cli.py:1-294; SURVEY next-3).

    python -m paper_1609_04567_b200.cli gol --n 128 --m 128 -p 4 --mode 1:n --csv out.csv
    python -m paper_1609_04567_b200.cli helmholtz --n 256 --m 256 --tol 1e-6
    python -m paper_1609_04567_b200.cli sobel --in lena.pgm --out edges.pgm
    python -m paper_1609_04567_b200.cli denoise --in noisy.pgm --out clean.pgm
    python -m paper_1609_04567_b200.cli denoise --frames 8 -w 4 --noise-level 0.1

Same commands, options, synthetic inputs, stdout lines, CSV rows and exit
status (0 ok, 1 run failure, 2 usage error) as the reference's `stencilkit`
command, so scripts driving it switch by changing the program name.  Every
run happens on the GPU; the reported wall_ms covers the pattern run only
(the reference's rule), never file IO or input synthesis.
"""

from __future__ import annotations

import argparse
import os
import sys
import time
from typing import Optional

import numpy as np

from .apps import (GolConfig, HelmholtzConfig, RestoreConfig, amf_detect, game_of_life,
                   helmholtz_solve, restore_regularize, salt_pepper, sobel_filter,
                   video_restore_pipeline)
from .bench import BenchRow, RunSpec, emit_csv
from .grid import Grid, GridError
from .partition import DeploymentMode
from .patterns import StencilError
from .pgm import read_pgm, write_pgm
from .streams import StreamError

# options every command takes: (flags, argparse keywords)
_SHARED = (
    (("-p", "--partitions"), dict(type=int, default=1, help="partitions per run (default 1)")),
    (("-w", "--width"), dict(type=int, default=1, help="stream farm width (default 1)")),
    (("--mode",), dict(choices=("1:1", "1:n"), default="1:1",
                       help="deployment: 1:1 whole-grid, 1:n split grid")),
    (("--seed",), dict(type=int, default=42, help="RNG seed for synthetic inputs (default 42)")),
    (("--csv",), dict(metavar="PATH", help="append a benchmark row to PATH")),
    (("--max-iters",), dict(type=int, default=None, help="iteration cap (app-specific default)")),
)
_N = (("--n",), dict(type=int, default=64, help="rows (default 64)"))
_M = (("--m",), dict(type=int, default=64, help="cols (default 64)"))


def synthetic_frame(rows: int, cols: int, shift: int) -> Grid:
    """The CLI's synthetic test frame (cli.py:187-191): (3r + 2c + 5 shift) mod 256."""
    r = np.arange(rows, dtype=np.int64)[:, None]
    c = np.arange(cols, dtype=np.int64)[None, :]
    return Grid.from_array((3 * r + 2 * c + 5 * shift) % 256)


def _rounded(g: Grid) -> Grid:
    """Restored (fp64) image -> the 8-bit image written out (cli.py:128-130)."""
    return Grid.from_array(np.clip(np.rint(g.to_array(dtype=np.float64)), 0, 255).astype(np.int64))


def _numbered_writer(directory: str, rounded: bool = True):
    """frameNNNN.pgm in call order (= stream order)."""
    os.makedirs(directory, exist_ok=True)
    seq = [0]

    def write(g: Grid) -> None:
        path = os.path.join(directory, f"frame{seq[0]:04d}.pgm")
        seq[0] += 1
        write_pgm(path, _rounded(g) if rounded else g)

    return write


class _Run:
    """Banner, timing and CSV row of one command."""

    def __init__(self, args, input_id: str):
        self.args, self.input_id = args, input_id
        print(f"{args.command} {input_id} p={args.partitions} w={args.width} "
              f"mode={args.mode} seed={args.seed}")

    def timed(self, fn, *a, **kw):
        t0 = time.perf_counter()
        res = fn(*a, **kw)
        self.wall_ms = (time.perf_counter() - t0) * 1e3
        return res

    def spec(self) -> RunSpec:
        a = self.args
        return RunSpec(app=a.command, input_id=self.input_id, partitions=a.partitions,
                       width=a.width, mode=a.mode, seed=a.seed)

    def csv_row(self, report) -> None:
        if self.args.csv:
            emit_csv([BenchRow.from_run(self.spec(), report, self.wall_ms)], self.args.csv)


def _mode(args) -> DeploymentMode:
    return DeploymentMode.parse(args.mode)


def cmd_gol(args) -> int:
    rng = np.random.default_rng(args.seed)
    soup = Grid.from_array((rng.random((args.n, args.m)) < 0.3).astype(np.int64))
    run = _Run(args, f"soup-{args.n}x{args.m}")
    board, rep = run.timed(game_of_life, soup,
                           config=GolConfig(rows=args.n, cols=args.m,
                                            steps=args.max_iters or 100),
                           partitions=args.partitions, mode=_mode(args))
    print(f"iterations={rep.iterations} liveness={rep.final_reduce} wall_ms={run.wall_ms:.3f}")
    if args.out:
        write_pgm(args.out, Grid.from_array(255 * board.to_array().astype(np.int64)))
    run.csv_row(rep)
    return 0


def cmd_helmholtz(args) -> int:
    n, m = args.n, args.m
    cfg = HelmholtzConfig(rows=n, cols=m, alpha=args.alpha, tol=args.tol,
                          max_iterations=args.max_iters or 10_000)
    run = _Run(args, f"unit-{n}x{m}")
    _u, rep = run.timed(helmholtz_solve, cfg, Grid.filled((n, m), 1.0),
                        partitions=args.partitions, mode=_mode(args))
    rms = (rep.final_reduce / (n * m)) ** 0.5
    print(f"iterations={rep.iterations} rms_step={rms:.3e} "
          f"{'exhausted' if rep.exhausted else 'converged'} wall_ms={run.wall_ms:.3f}")
    run.csv_row(rep)
    return 0


def cmd_sobel(args) -> int:
    img = read_pgm(args.infile)
    run = _Run(args, args.infile.rsplit("/", 1)[-1])
    edges, rep = run.timed(sobel_filter, img, partitions=args.partitions, mode=_mode(args),
                           with_report=True)
    print(f"pixel_sum={rep.final_reduce} wall_ms={run.wall_ms:.3f}")
    if args.out:
        write_pgm(args.out, edges)
    run.csv_row(rep)
    return 0


def _denoise_frames(args, cfg) -> int:
    src = str(args.frames)
    if src.isdigit():
        count = int(src)
        if count < 1:
            raise GridError(f"--frames count must be >= 1, got {args.frames}")
        level = 0.1 if args.noise_level is None else args.noise_level
        frames = [salt_pepper(synthetic_frame(args.n, args.m, i), level, seed=args.seed + i)[0]
                  for i in range(count)]
        input_id = f"frames{count}-{args.n}x{args.m}"
    else:
        names = sorted(p for p in os.listdir(src) if p.endswith(".pgm"))
        if not names:
            raise GridError(f"no .pgm frames in {src!r}")
        frames = [read_pgm(os.path.join(src, p)) for p in names]
        input_id = os.path.basename(os.path.normpath(src))
    writer = _numbered_writer(args.out) if args.out else None
    masks = _numbered_writer(args.noise_map_out) if args.noise_map_out else None
    run = _Run(args, input_id)
    rep = run.timed(video_restore_pipeline, frames, width=args.width,
                    partitions=args.partitions, mode=_mode(args), cfg=cfg, writer=writer,
                    mask_writer=masks)
    print(f"frames={rep.items_out} failures={len(rep.failures)} wall_ms={run.wall_ms:.3f}")
    if args.csv:
        s = run.spec()
        emit_csv([BenchRow(s.app, s.input_id, s.partitions, s.width, s.mode.value, s.seed,
                           rep.items_out, run.wall_ms, 0, 0, 0, 0.0)], args.csv)
    return 1 if rep.failures else 0


def cmd_denoise(args) -> int:
    cap = args.max_iters or 100
    cfg = RestoreConfig(max_iterations=cap) if args.tol is None else \
        RestoreConfig(tol=args.tol, max_iterations=cap)
    if args.frames is not None:
        return _denoise_frames(args, cfg)
    if args.infile:
        img, input_id = read_pgm(args.infile), args.infile.rsplit("/", 1)[-1]
        level = args.noise_level or 0.0
    else:
        img, input_id = synthetic_frame(args.n, args.m, 0), f"synthetic-{args.n}x{args.m}"
        level = 0.1 if args.noise_level is None else args.noise_level
    if level > 0:
        img = salt_pepper(img, level, seed=args.seed)[0]
    run = _Run(args, input_id)
    mode = _mode(args)

    def both():
        mask = amf_detect(img, wmax=cfg.amf_wmax, partitions=args.partitions, mode=mode)
        restored, rep = restore_regularize(img, mask, cfg, partitions=args.partitions, mode=mode)
        return mask, restored, rep

    mask, restored, rep = run.timed(both)
    flagged = int(mask.to_array().sum())
    print(f"flagged={flagged} iterations={rep.iterations} "
          f"{'exhausted' if rep.exhausted else 'converged'} wall_ms={run.wall_ms:.3f}")
    if args.out:
        write_pgm(args.out, _rounded(restored))
    run.csv_row(rep)
    return 0


_COMMANDS = {
    "gol": ("Game of Life on a random soup", cmd_gol,
            [_N, _M, (("--out",), dict(help="write the final board as PGM"))]),
    "helmholtz": ("Jacobi Helmholtz solve, unit forcing", cmd_helmholtz,
                  [_N, _M,
                   (("--alpha",), dict(type=float, default=1.0,
                                       help="Helmholtz coefficient (default 1.0)")),
                   (("--tol",), dict(type=float, default=1e-6,
                                     help="RMS step-size tolerance (default 1e-6)"))]),
    "sobel": ("Sobel edge detection on a PGM image", cmd_sobel,
              [(("--in",), dict(dest="infile", required=True, help="input PGM")),
               (("--out",), dict(help="write the edge map as PGM"))]),
    "denoise": ("impulse-noise removal, image or frames", cmd_denoise,
                [(("--in",), dict(dest="infile", help="input PGM (else synthetic)")),
                 (("--out",), dict(help="write the restored image as PGM")),
                 (("--n",), dict(type=int, default=64, help="synthetic rows (default 64)")),
                 (("--m",), dict(type=int, default=64, help="synthetic cols (default 64)")),
                 (("--frames",), dict(default=None, help="stream a directory of PGM frames (or a "
                                                         "count of synthetic frames) instead of a "
                                                         "single image")),
                 (("--noise-map-out",), dict(metavar="DIR", help="with --frames: write per-frame "
                                                                 "noise maps here")),
                 (("--noise-level",), dict(type=float, default=None,
                                           help="salt-and-pepper fraction to inject (default 0.1 "
                                                "synthetic, 0 for --in)")),
                 (("--tol",), dict(type=float, default=None,
                                   help="restoration tolerance (default 0.02)"))]),
}


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="stencilkit",
                                 description="iterative stencil apps on partitioned grids "
                                             "(B200 engine)")
    sub = ap.add_subparsers(dest="command", required=True)
    for name, (helptext, fn, own) in _COMMANDS.items():
        p = sub.add_parser(name, help=helptext)
        for flags, kw in _SHARED + tuple(own):
            p.add_argument(*flags, **kw)
        p.set_defaults(func=fn)
    return ap


def main(argv: Optional[list] = None) -> int:
    ap = build_parser()
    args = ap.parse_args(argv)
    if args.mode == "1:n" and args.partitions < 2:
        ap.error("mode 1:n needs --partitions >= 2")
    try:
        return args.func(args)
    except (GridError, StencilError, StreamError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())

"""PGM frames either side of the stream (reference: pgm.py:1-132; SURVEY next-3).

Same contract as the reference's read_pgm / write_pgm: P2 (ASCII) and P5
(binary) graymaps with maxval <= 255, whitespace and `#` comments in the
header (and between P2 samples), exactly one whitespace byte between the P5
header and its raster, and a PgmError (a GridError) carrying the byte
offset where parsing gave up.

What differs is the representation: the raster is decoded with numpy into
one uint8 array (no per-pixel Python objects), so a frame can go to the
device as one 1-byte-per-pixel upload; `Grid.data` still yields the same
list of ints the reference returns.
"""

from __future__ import annotations

import os
import re
from typing import Union

import numpy as np

from .grid import Grid, GridError

_WS = b" \t\r\n\x0b\x0c"
# a sample / header token, or a comment running to the end of its line
_TOKENS = re.compile(rb"#[^\r\n]*|[^ \t\r\n\x0b\x0c#]+")


class PgmError(GridError):
    """Malformed PGM input; `offset` is the byte position of the problem."""

    def __init__(self, message: str, offset: int):
        super().__init__(f"{message} (byte offset {offset})")
        self.offset = offset


class _Header:
    """Reads the header fields one token at a time, remembering offsets."""

    def __init__(self, data: bytes):
        self.data = data
        self.pos = 0
        self.tok_at = 0

    def next(self, what: str) -> bytes:
        n = len(self.data)
        while True:
            m = _TOKENS.search(self.data, self.pos)
            if m is None:
                # only separators (and comments) left
                raise PgmError(f"unexpected end of file reading {what}", n)
            if m.group().startswith(b"#"):
                self.pos = m.end()
                continue
            # anything between pos and the match must be whitespace
            self.tok_at, self.pos = m.start(), m.end()
            return m.group()

    def number(self, what: str) -> int:
        tok = self.next(what)
        try:
            return int(tok)
        except ValueError:
            raise PgmError(f"expected integer for {what}, got {tok!r}", self.tok_at) from None


def read_pgm(path: Union[str, os.PathLike]) -> Grid:
    """Load a P2 or P5 graymap as a 2D grid of ints in [0, maxval]
    (pgm.py:63-104), stored as uint8."""
    with open(path, "rb") as fh:
        data = fh.read()
    hd = _Header(data)
    magic = hd.next("magic number")
    if magic not in (b"P2", b"P5"):
        raise PgmError(f"not a PGM file, magic {magic!r}", 0)
    width = hd.number("width")
    height = hd.number("height")
    maxval = hd.number("maxval")
    if width <= 0 or height <= 0:
        raise PgmError(f"bad dimensions {width}x{height}", hd.pos)
    if not 0 < maxval <= 255:
        raise PgmError(f"unsupported maxval {maxval}", hd.pos)
    count = width * height
    if magic == b"P5":
        if hd.pos >= len(data) or data[hd.pos] not in b" \t\r\n":
            raise PgmError("missing whitespace after maxval", hd.pos)
        start = hd.pos + 1
        if len(data) - start < count:
            raise PgmError(f"raster truncated: expected {count} bytes, found {len(data) - start}",
                           len(data))
        raster = np.frombuffer(data, dtype=np.uint8, count=count, offset=start)
        if maxval < 255:
            bad = np.flatnonzero(raster > maxval)
            if bad.size:
                i = int(bad[0])
                raise PgmError(f"pixel value {int(raster[i])} exceeds maxval {maxval}", start + i)
        return Grid((height, width), raster.reshape(height, width).copy())
    # P2: `count` integer tokens, comments allowed in between
    out = np.empty(count, dtype=np.uint8)
    k = 0
    for m in _TOKENS.finditer(data, hd.pos):
        if k == count:
            break
        tok = m.group()
        if tok.startswith(b"#"):
            continue
        try:
            v = int(tok)
        except ValueError:
            raise PgmError(f"expected integer for pixel value, got {tok!r}", m.start()) from None
        if not 0 <= v <= maxval:
            raise PgmError(f"pixel value {v} exceeds maxval {maxval}", m.start())
        out[k] = v
        k += 1
    if k < count:
        raise PgmError("unexpected end of file reading pixel value", len(data))
    return Grid((height, width), out.reshape(height, width))


def _pixels(img: Grid, maxval: int) -> np.ndarray:
    """The grid's values as uint8, each checked to be an integer in
    [0, maxval] (first offender reported as the reference does)."""
    a = np.asarray(img.to_array())
    if a.dtype == object:
        flat = list(a.ravel())
        for v in flat:
            iv = int(v)
            if iv != v or not 0 <= iv <= maxval:
                raise GridError(f"pixel value {v!r} not an integer in [0, {maxval}]")
        return np.asarray(flat, dtype=np.int64).astype(np.uint8).reshape(a.shape)
    flat = a.ravel()
    if a.dtype.kind == "b":
        ok = np.ones(flat.shape, bool) if maxval >= 1 else ~flat
    elif a.dtype.kind in "iu":
        ok = (flat >= 0) & (flat <= maxval)
    else:
        with np.errstate(invalid="ignore"):
            ok = (flat == np.floor(flat)) & (flat >= 0) & (flat <= maxval)
    if not ok.all():
        v = flat[int(np.flatnonzero(~ok)[0])].item()
        raise GridError(f"pixel value {v!r} not an integer in [0, {maxval}]")
    return flat.astype(np.uint8).reshape(a.shape)


def write_pgm(path: Union[str, os.PathLike], img: Grid, *,
              binary: bool = True, maxval: int = 255) -> None:
    """Write a 2D grid of ints in [0, maxval] as P5 (or P2 when binary=False)
    (pgm.py:107-132); device grids are read back once."""
    if img.ndim != 2:
        raise GridError("PGM output expects a 2D grid")
    if not 0 < maxval <= 255:
        raise GridError(f"unsupported maxval {maxval}")
    rows, cols = img.dims
    px = _pixels(img, maxval)
    head = f"P5\n{cols} {rows}\n{maxval}\n" if binary else f"P2\n{cols} {rows}\n{maxval}\n"
    if binary:
        with open(path, "wb") as fh:
            fh.write(head.encode("ascii"))
            fh.write(px.tobytes())
        return
    body = "".join(" ".join(map(str, row.tolist())) + "\n" for row in px)
    with open(path, "w", encoding="ascii") as fh:
        fh.write(head + body)

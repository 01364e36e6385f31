"""Band text I/O: the reference's fixture format
(banded.cpp:192-225, banded.hpp:181-185), for interchange with the reference
tools and tests.

Format: a header ``band n lower upper`` and then the ``lower + upper + 1``
storage rows, each the ``n`` values of that storage row in ``%.17g``
(round-trips IEEE doubles exactly), space separated.  Corner cells (storage
cells with no matrix entry) must be zero; reading rejects anything else with
:class:`MalformedInput`, as the reference does.  A batch is written as
consecutive blocks, one per matrix (a single block is exactly the
reference's file).  Host-side only: this is the file format, not a compute
path.
"""
from __future__ import annotations

import io
import os

import numpy as np

from .api import BandgmError


class MalformedInput(BandgmError):
    """errors.hpp:126-128"""


def _corner_mask(n: int, lower: int, upper: int) -> np.ndarray:
    """(n, w) mask of storage cells outside the matrix: row r of column j holds i = j + r - upper."""
    r = np.arange(lower + upper + 1)[None, :]
    i = np.arange(n)[:, None] + r - upper
    return (i < 0) | (i >= n)


def dumps(arr, lower: int, upper: int) -> str:
    """write_band_text (banded.cpp:192-202) of one matrix; arr[j, r] = storage row r of column j."""
    a = np.asarray(arr, dtype=np.float64)
    n, w = a.shape
    if w != lower + upper + 1:
        raise MalformedInput("band text: storage rows do not match the band")
    out = [f"band {n} {lower} {upper}\n"]
    for r in range(w):
        out.append(" ".join("%.17g" % v for v in a[:, r]) + "\n")
    return "".join(out)


def _read_one(tok, pos: int):
    if pos + 4 > len(tok) or tok[pos] != "band":
        raise MalformedInput("band text: expected header 'band n lower upper'")
    try:
        n, lo, up = (int(t) for t in tok[pos + 1:pos + 4])
    except ValueError:
        raise MalformedInput("band text: expected header 'band n lower upper'") from None
    if n < 0 or lo < 0 or up < 0:
        raise MalformedInput("band text: negative dimension")
    w = lo + up + 1
    pos += 4
    if pos + w * n > len(tok):
        raise MalformedInput("band text: truncated value block")
    try:
        vals = np.array([float(t) for t in tok[pos:pos + w * n]], dtype=np.float64)
    except ValueError:
        raise MalformedInput("band text: truncated value block") from None
    a = vals.reshape(w, n).T.copy()
    if np.any(a[_corner_mask(n, lo, up)] != 0.0):
        raise MalformedInput("band text: nonzero corner cell")
    return a, lo, up, pos + w * n


def loads(text: str):
    """read_band_text (banded.cpp:204-225) of one matrix -> (arr (n, w), lower, upper)."""
    tok = text.split()
    a, lo, up, _ = _read_one(tok, 0)
    return a, lo, up


def loads_all(text: str):
    """All consecutive blocks -> (arr (B, n, w), lower, upper); every block must share n and the band."""
    tok = text.split()
    pos, mats, shape = 0, [], None
    while pos < len(tok):
        a, lo, up, pos = _read_one(tok, pos)
        if shape is None:
            shape = (a.shape[0], lo, up)
        elif shape != (a.shape[0], lo, up):
            raise MalformedInput("band text: blocks of one batch must share n and the band")
        mats.append(a)
    if not mats:
        raise MalformedInput("band text: expected header 'band n lower upper'")
    return np.stack(mats), shape[1], shape[2]


def write_band_text_file(path: str | os.PathLike, bands_or_arr, lower: int | None = None,
                         upper: int | None = None) -> None:
    """write_band_text_file (banded.cpp:227-231) for a device Bands batch or a
    host array ((n, w) or (B, n, w))."""
    if hasattr(bands_or_arr, "numpy") and hasattr(bands_or_arr, "lower"):
        arr, lower, upper = bands_or_arr.numpy(), bands_or_arr.lower, bands_or_arr.upper
    else:
        arr = np.asarray(bands_or_arr, dtype=np.float64)
    if arr.ndim == 2:
        arr = arr[None]
    with open(path, "w") as f:
        for a in arr:
            f.write(dumps(a, lower, upper))


def read_band_text_file(path: str | os.PathLike, tile: int | None = None, device=None):
    """read_band_text_file (banded.cpp:233-237): (B, n, w) host array with its
    band, or a device Bands batch when ``tile`` is given."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise MalformedInput(f"cannot open '{path}'") from None
    arr, lo, up = loads_all(text)
    if tile is None:
        return arr, lo, up
    from .api import Bands
    return Bands.from_reference(arr, lo, up, tile=tile, device=device)


__all__ = ["MalformedInput", "dumps", "loads", "loads_all", "write_band_text_file", "read_band_text_file",
           "io"]

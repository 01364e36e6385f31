"""Band text I/O (banded.cpp:192-237): the Python writer is byte-identical to
the verbatim reference writer (oracle/_ref), round trips are bit-exact, and
the reference's malformed-input cases raise MalformedInput
(test_banded.cpp:131-160).  Host-only: runs without a GPU."""
import ctypes as C

import numpy as np
import pytest

import oracle as orc
from paper_1902_10078_b200 import bandio
from tests import common as cm


def _ref_text(a, lo, up):
    lib = C.CDLL(orc.LIB_PATHS["reference"][0])
    f = lib.ref_write_band_text
    f.restype = C.c_longlong
    n = a.shape[0]
    buf = C.create_string_buffer(64 * (n + 4) * (lo + up + 1) + 64)
    k = f(C.c_int64(n), C.c_int64(lo), C.c_int64(up), np.ascontiguousarray(a).ctypes.data_as(C.POINTER(C.c_double)),
          buf, C.c_longlong(len(buf)))
    assert k >= 0
    return buf.value.decode()


def test_round_trip_and_reference_bytes():
    rng = np.random.default_rng(15)
    for _ in range(10):  # test_banded.cpp:135-150
        n = int(rng.integers(1, 26))
        lo, up = min(int(rng.integers(0, 4)), n - 1), min(int(rng.integers(0, 4)), n - 1)
        a = cm.random_band(rng, 1, n, lo, up)[0] * 1e-7
        text = bandio.dumps(a, lo, up)
        back, blo, bup = bandio.loads(text)
        assert (blo, bup) == (lo, up)
        assert np.array_equal(back.view(np.uint64), a.view(np.uint64))
        assert bandio.dumps(back, lo, up) == text
        if orc.available("reference"):
            assert text == _ref_text(a, lo, up)


def test_malformed_inputs():
    for bad in ("bands 3 1 1\n", "band 3 1 1\n0 1 2\n3 4", "band 2 0 1\n9 1\n2 3\n", "band -1 0 0\n", ""):
        with pytest.raises(bandio.MalformedInput):
            bandio.loads_all(bad)


def test_batch_file(tmp_path):
    rng = np.random.default_rng(3)
    a = cm.random_band(rng, 4, 17, 2, 1)
    p = tmp_path / "batch.band"
    bandio.write_band_text_file(p, a, 2, 1)
    back, lo, up = bandio.read_band_text_file(p)
    assert (lo, up) == (2, 1) and np.array_equal(back, a)
    with pytest.raises(bandio.MalformedInput):
        bandio.read_band_text_file(tmp_path / "missing.band")

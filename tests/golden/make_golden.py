"""Regenerates tests/golden/golden_v1.npz from the reference compiled verbatim.

    python -m tests.golden.make_golden

Needs oracle/_ref/libbandgm_ref.so (built by `make -C oracle` where
/root/reference exists).  The fixture is committed; the GPU box never runs
this script.
"""
import os

import numpy as np

import oracle as orc
from tests.golden.cases import CASES, run_case

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_v1.npz")


def main():
    ref = orc.Oracle("reference")
    arrays = {}
    for name in CASES:
        for key, val in run_case(name, ref).items():
            arrays[f"{name}/{key}"] = np.asarray(val)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT}: {len(arrays)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()

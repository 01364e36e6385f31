"""CPU: the C-ABI library loads and exports every symbol include/bandgm_b200.h
declares, and carries sm_100a code.  No compute calls (no GPU here)."""
import ctypes
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bandgm_b200.h")
LIB = os.path.join(ROOT, "paper_1902_10078_b200", "libbandgm_b200.so")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(bgm_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1902_10078_b200")], check=True)
    return ctypes.CDLL(LIB)


def test_every_declared_symbol_is_exported(lib):
    names = declared()
    assert len(names) >= 24
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_host_only_entry_points(lib):
    assert lib.bgm_abi_version() == 1
    lib.bgm_status_name.restype = ctypes.c_char_p
    assert lib.bgm_status_name(1) == b"NotPositiveDefinite"
    # argument validation runs on the host: a bad tile is rejected before any launch
    from paper_1902_10078_b200.api import _Band
    bad = _Band(None, 1, 4, 1, 0, 7, 0)
    assert lib.bgm_cholesky(bad, bad, None, None, None) == 5  # BGM_ERR_ARG


@pytest.mark.skipif(shutil.which("cuobjdump") is None and not os.path.exists("/usr/local/cuda/bin/cuobjdump"),
                    reason="cuobjdump missing")
def test_library_targets_sm100a():
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([tool, "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out

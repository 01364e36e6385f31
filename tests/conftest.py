import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: full-size configuration checks")


@pytest.fixture(scope="session")
def oracle():
    """The plain-C restatement (always built)."""
    import oracle as orc

    if not orc.available("restatement"):
        orc.build(reference=False)
    return orc.Oracle("restatement")


@pytest.fixture(scope="session")
def reference():
    """The verbatim-compiled reference, when its prebuilt .so is present."""
    import oracle as orc

    if not orc.available("reference"):
        try:
            orc.build(reference=True)
        except Exception:
            pass
    if not orc.available("reference"):
        pytest.skip("oracle/_ref not built (no /root/reference here and no prebuilt .so)")
    return orc.Oracle("reference")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1902_10078_b200 as bgm

    bgm.library()
    return bgm

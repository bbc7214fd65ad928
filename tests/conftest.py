import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built librt_b200.so")
    config.addinivalue_line("markers", "slow: long-running")



@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def cornell_oracle(oracle_mod):
    from paper_2603_00292_b200 import scenes
    return oracle_mod.scene_from_description(scenes.cornell_description())


@pytest.fixture(scope="session")
def reference():
    """The reference package itself (build container only; never on the GPU box)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference not present (GPU box)")
    from rt_helpers import import_reference
    return import_reference()


@pytest.fixture(scope="session")
def native():
    """The CUDA C-ABI library on a real GPU; fails loudly if missing on a GPU box."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_00292_b200 import _native
    return _native.lib()

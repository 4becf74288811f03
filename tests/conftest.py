import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")
    config.addinivalue_line("markers", "slow: full-size configs (minutes)")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build_lib()
    return oracle


def build_native():
    """Compile libwt.so (nvcc, sm_100a) without importing the package first."""
    import importlib.util
    path = os.path.join(ROOT, "paper_1610_05994_b200", "buildlib.py")
    spec = importlib.util.spec_from_file_location("wt_buildlib", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.build()

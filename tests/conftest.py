import sys
from pathlib import Path


ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))



def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a) and libstl_b200.so")


import pytest  # noqa: E402


@pytest.fixture(scope="session")
def lib_path():
    return ROOT / "paper_2503_12211_b200" / "libstl_b200.so"

import os
import sys
import tempfile
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))
# compiled-dynamics cache of this test session (not the user's ~/.cache)
os.environ.setdefault("GM_JIT_CACHE", tempfile.mkdtemp(prefix="gm_jit_cache_"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: larger parity sizes")

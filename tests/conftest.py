import os
import sys
from pathlib import Path

import pytest

# thread ranks sharing one GPU put 2 streams per rank behind stream-side
# waits: give every stream its own hardware queue (set before CUDA init)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs")


@pytest.fixture(scope="session")
def golden_kernels():
    import numpy as np
    return dict(np.load(GOLDEN / "golden_kernels.npz"))


@pytest.fixture(scope="session")
def golden_strategies():
    import numpy as np
    return dict(np.load(GOLDEN / "golden_strategies.npz"))


@pytest.fixture(scope="session")
def golden_c1():
    import numpy as np
    return dict(np.load(GOLDEN / "golden_c1.npz"))


@pytest.fixture(scope="session")
def golden_mllm_ca():
    import numpy as np
    return dict(np.load(GOLDEN / "golden_mllm_ca.npz"))

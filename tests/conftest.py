import os
import sys

# In-process groups on ONE GPU (bcgs_create_local_p2p) run each rank's kernels concurrently
# with the others' spin-waiting kernels; lazily loading a kernel module at its first launch
# can stall behind those waits.  Load every module when the CUDA context is created.
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (large grids)")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.lib()
    return oracle

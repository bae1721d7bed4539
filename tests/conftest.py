import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    # the C restatement is plain C: build it on demand (gcc exists here and on the GPU box)
    so = os.path.join(ROOT, "oracle", "_build", "libsemwarm_oracle.so")
    if not os.path.exists(so):
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"])


def have_ref() -> bool:
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libsemwarm_ref.so"))


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    if not have_ref():
        pytest.skip("compiled reference (oracle/_ref) not present")
    import oracle
    return oracle.Ref()


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return {n[:-4]: np.load(os.path.join(GOLDEN, n)) for n in os.listdir(GOLDEN)
            if n.endswith(".npz")}

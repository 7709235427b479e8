import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")
    config.addinivalue_line("markers", "ref: needs oracle/_ref (the compiled reference)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    # native artefacts are built in-tree; rebuild only if missing
    from paper_2603_09983_b200 import build as b
    if not os.path.exists(b.LIB):
        b.build()
    import oracle as O
    if not os.path.exists(O._ORC_PATH):
        O.build()
    yield


def ref_or_skip():
    import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")

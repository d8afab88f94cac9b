import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
for p in (ROOT, TESTS, os.path.join(TESTS, "golden")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "ref: needs the reference compiled in place (oracle/_ref)")


def pytest_collection_modifyitems(config, items):
    import _oracle

    if not _oracle.have_ref():
        skip = pytest.mark.skip(reason="oracle/_ref/libpcvref.so not built (needs /root/reference)")
        for item in items:
            if "ref" in item.keywords:
                item.add_marker(skip)

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "ref: needs oracle/_ref/libweft_ref.so (the compiled reference)")


def pytest_collection_modifyitems(config, items):
    from oracle_bindings import REF

    skip_ref = pytest.mark.skip(reason="oracle/_ref not built (needs /root/reference at build time)")
    for item in items:
        if "ref" in item.keywords and REF is None:
            item.add_marker(skip_ref)
